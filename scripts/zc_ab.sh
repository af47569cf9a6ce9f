# zero-copy host path: parity + e2e A/B (MC_NO_ZERO_COPY=1 = chunked copy pipeline)
timeout 900 python -m pytest tests/test_gpu_conv.py -q -x 2>&1 | tail -1
MC_BULK_OUT=1 timeout 900 python -m pytest tests/test_gpu_conv.py -q -x 2>&1 | tail -1
timeout 200 python scripts/zc_probe2.py
for v in "" 1; do
  echo "== MC_NO_ZERO_COPY=$v"
  for c in 2 3 1; do
    MC_NO_ZERO_COPY=$v python bench.py --config $c --steps 10 --warmup 4 --ref-seconds 0.1 > gpurun_out/zc$c.json 2>&1; python scripts/summ.py gpurun_out/zc$c.json
  done
done
echo "== MC_BULK_OUT=1 (device path)"
MC_BULK_OUT=1 python bench.py --config 2 --steps 20 --warmup 4 --ref-seconds 0.1 > gpurun_out/zcb2.json 2>&1; python scripts/summ.py gpurun_out/zcb2.json
