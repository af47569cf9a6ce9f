# A/B of the four-step row length (MC_FOURSTEP_KC=11 vs the default 12) on configs 4 and 5
MC_FOURSTEP_KC=11 timeout 600 python -m pytest tests/test_gpu_fourstep.py -q -k "cfg4 or cfg5" 2>&1 | tail -2
for rep in 1 2; do
  for kc in 12 11; do
    for c in 5 4; do
      MC_FOURSTEP_KC=$kc python bench.py --config $c --configs head --steps 20 --ref-seconds 0.1 > gpurun_out/kc_${kc}_cfg${c}.json 2>/dev/null
      python - <<PY
import json; d=json.load(open("gpurun_out/kc_${kc}_cfg${c}.json"))
print("KC=$kc cfg$c rep$rep", round(d["ms_per_step"]*1e3,1), "us", d["clocks"]["sm_mhz"])
PY
    done
  done
done
