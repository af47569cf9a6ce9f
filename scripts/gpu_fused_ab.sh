# fused-kernel check after a change: GPU parity tests, then cfg2/cfg3/cfg1 benches
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 2 3 1; do
  python bench.py --config $c --steps 10 --warmup 3 --ref-seconds 1 > gpurun_out/ab_cfg$c.json 2> gpurun_out/ab_cfg$c.err
  python scripts/summ.py gpurun_out/ab_cfg$c.json
done
