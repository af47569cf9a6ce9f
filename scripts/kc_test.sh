timeout 600 python -m pytest tests/test_gpu_fourstep.py -q -x 2>&1 | tail -1
for kc in 12 13; do
  echo "== KC $kc"; MC_FOURSTEP_KC=$kc python bench.py --config 4 --steps 10 --warmup 3 --ref-seconds 0.1 > gpurun_out/kc.json 2>&1 && python scripts/summ.py gpurun_out/kc.json
  MC_FOURSTEP_KC=$kc python bench.py --config 5 --steps 10 --warmup 3 --ref-seconds 0.1 > gpurun_out/kc5.json 2>&1 && python scripts/summ.py gpurun_out/kc5.json
done
