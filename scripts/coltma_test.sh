timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_split.py -q -x 2>&1 | tail -1
for v in "" 1; do
  echo "== MC_NO_COL_TMA=$v"
  MC_NO_COL_TMA=$v python bench.py --config 4 --steps 10 --warmup 3 --ref-seconds 0.1 > gpurun_out/t4.json 2>&1; python scripts/summ.py gpurun_out/t4.json
  MC_NO_COL_TMA=$v python bench.py --config 5 --steps 10 --warmup 3 --ref-seconds 0.1 > gpurun_out/t5.json 2>&1; python scripts/summ.py gpurun_out/t5.json
done
