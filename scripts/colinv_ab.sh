# A/B of the async-copy inverse column pass (default on; MC_NO_COL_INV_ASYNC=1 disables) on cfg4/cfg5 + launch lists
timeout 900 python -m pytest tests/test_gpu_fourstep.py -q -x 2>&1 | tail -1
MC_NO_COL_INV_ASYNC=1 timeout 900 python -m pytest tests/test_gpu_fourstep.py -q -x 2>&1 | tail -1
for v in "" 1; do
  echo "== MC_NO_COL_INV_ASYNC=$v"
  for c in 4 5; do
    MC_NO_COL_INV_ASYNC=$v python bench.py --config $c --steps 10 --warmup 4 --ref-seconds 0.1 > gpurun_out/ci$c.json 2>&1; python scripts/summ.py gpurun_out/ci$c.json
  done
done
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -c 12 --csv --log-file gpurun_out/launches_ci_async.csv python bench.py --config 4 --steps 2 --warmup 3 --ref-seconds 0.1 > /dev/null 2>&1
echo "ncu rc=$?"
