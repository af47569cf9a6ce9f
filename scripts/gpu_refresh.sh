# round-end evidence refresh for HEAD: launch list of the default bench (cfg2),
# ncu --set full of the cfg2 fused kernel, step launch lists with DRAM bytes for
# configs 1, 3, 4, 5, and the multi-rank bench path (2 ranks, gloo host collectives)
TAG=${1:-head}
python bench.py --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/rf_plain.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg2_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/rf_ncu1.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:conv_small -s 2 -c 1 -o gpurun_out/prof_cfg2_$TAG \
  python bench.py --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/rf_ncu2.log 2>&1; echo "full rc=$?"
for c in 1 3 4 5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -c 80 --csv \
    --log-file gpurun_out/traffic_cfg${c}_$TAG.csv python bench.py --config $c --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/rf_t$c.log 2>&1; echo "traffic cfg$c rc=$?"
done
timeout 600 bash scripts/gpu_multirank.sh > gpurun_out/rf_multirank.log 2>&1; echo "multirank rc=$?"; tail -5 gpurun_out/rf_multirank.log
