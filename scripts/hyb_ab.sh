timeout 900 python -m pytest tests/test_gpu_conv.py -q -x 2>&1 | tail -1
python scripts/e2e_test.py
for c in 2 3 1; do
  python bench.py --config $c --steps 10 --warmup 4 --ref-seconds 0.1 > gpurun_out/hy$c.json 2>&1; python scripts/summ.py gpurun_out/hy$c.json
done
