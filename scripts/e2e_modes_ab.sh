for rep in 1 2; do
for m in zc "in 4" "in 8" "in 16" "in 32" "ce 4" "ce 8"; do
  set -- $m
  MC_HOST_MODE=$1 MC_STREAM_IN_CHUNKS=${2:-32} MC_CE_CHUNKS=${2:-32} python bench.py --config 2 --configs head --steps 20 --warmup 5 --ref-seconds 0.1 > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo -n "rep$rep mode=$m: "; python scripts/summ.py gpurun_out/ab.json
done; done
