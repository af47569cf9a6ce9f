# refresh cfg4/cfg5 bench lines + launch lists + one full capture of the TMA column kernel
set -x
for c in 4 5; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; python scripts/summ.py gpurun_out/bench_cfg$c.json
done
bash scripts/gpu_launches.sh 4 b
bash scripts/gpu_launches.sh 5 b
ncu --set full --clock-control none --import-source on -k regex:col_fwd_tma -s 4 -c 1 -o gpurun_out/prof_cfg4_colfwd_tma python bench.py --config 4 --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
