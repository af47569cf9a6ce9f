# quick GPU check: parity tests + the three fused-kernel benches (no profiler)
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 --ref-seconds 1 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --config 1 --steps 20 --warmup 3 --ref-seconds 1 > gpurun_out/bench_cfg1.json 2>&1
python bench.py --config 3 --steps 5 --warmup 3 --ref-seconds 1 > gpurun_out/bench_cfg3.json 2>&1
for c in 2 1 3; do python -c "
import json; d=json.load(open('gpurun_out/bench_cfg$c.json'))
print('cfg$c', round(d['value']), d['unit'], 'kernel_ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']), 'clk', d['clocks'])
"; done
python bench.py --config 4 --steps 5 --warmup 3 --ref-seconds 1 > gpurun_out/bench_cfg4.json 2>&1
python bench.py --config 5 --steps 5 --warmup 3 --ref-seconds 1 > gpurun_out/bench_cfg5.json 2>&1
