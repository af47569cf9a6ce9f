# compute-sanitizer racecheck / synccheck / memcheck over every shared-memory
# and async-copy kernel (scripts/sanitize_cases.py), logs to gpurun_out/sanitize/
mkdir -p gpurun_out/sanitize
cases="fused_tma fused_small fused_host fourstep rowprefetch three_primes transforms"
for tool in memcheck racecheck synccheck; do
  for c in $cases; do
    env=""
    [ "$c" = rowprefetch ] && env="MC_ROW_PREFETCH=1"
    [ "$c" = fourstep ] && env="MC_ROW_PREFETCH=0"
    timeout 900 env $env compute-sanitizer --tool $tool --error-exitcode 99 \
        --log-file gpurun_out/sanitize/${tool}_${c}.log python scripts/sanitize_cases.py $c \
        > gpurun_out/sanitize/${tool}_${c}.out 2>&1
    echo "$tool $c rc=$? $(tail -1 gpurun_out/sanitize/${tool}_${c}.log)"
  done
done | tee gpurun_out/sanitize/summary.txt
