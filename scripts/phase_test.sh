for d in 0 300 600 1000 2000 4000; do
  echo "== delay $d"; MC_PHASE_NS=$d python bench.py --steps 30 --warmup 5 --ref-seconds 0.2 > gpurun_out/ph.json 2>&1 && python scripts/summ.py gpurun_out/ph.json
done
