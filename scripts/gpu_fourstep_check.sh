# four-step / three-primes: GPU tests, bench lines for configs 4 and 5, launch lists
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2; do for c in 5 4; do
  python bench.py --config $c --configs head --steps 20 --ref-seconds 0.1 > gpurun_out/b_cfg$c.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b_cfg$c.json'))
print('cfg$c rep$rep', round(d['ms_per_step']*1e3,1), 'us', d['clocks']['sm_mhz'], 'launches', d['gpu_launches'])"
done; done
for c in 5 4; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg${c}_r2.csv python bench.py --config $c --configs head --steps 2 --warmup 3 --ref-seconds 0.1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_cfg${c}_r2.csv | grep -v "at::\|gen_kernel"
done
