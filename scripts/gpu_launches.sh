# launch list (per-kernel device times) for a config: bash scripts/gpu_launches.sh <cfg> <tag>
CFG=${1:-4}; TAG=${2:-x}
python bench.py --config $CFG --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/plain_l$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -c 80 --csv --log-file gpurun_out/launches_cfg${CFG}_$TAG.csv python bench.py --config $CFG --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/ncu_l$TAG.log 2>&1
echo "rc=$?"
