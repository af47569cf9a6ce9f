set -x
python bench.py --steps 10 --warmup 3 --ref-seconds 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --config 1 --steps 20 --warmup 3 --ref-seconds 2 > gpurun_out/bench_cfg1.json 2>&1
python bench.py --config 3 --steps 5 --warmup 3 --ref-seconds 3 > gpurun_out/bench_cfg3.json 2>&1
python bench.py --steps 2 --warmup 3 --ref-seconds 0.2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --ref-seconds 0.2 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_small -s 2 -c 1 -o gpurun_out/prof_cfg2 python bench.py --steps 2 --warmup 3 --ref-seconds 0.2 > gpurun_out/ncu_full.log 2>&1
echo done
