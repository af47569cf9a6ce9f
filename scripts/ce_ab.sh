# e2e host modes A/B: default vs copy-engine whole-batch pipeline (MC_HOST_MODE=ce) at several chunk counts
for rep in 1 2; do
  python bench.py --config 2 --steps 10 --warmup 3 --ref-seconds 0.1 > gpurun_out/ce.json 2>&1; echo -n "rep$rep default cfg2: "; python scripts/summ.py gpurun_out/ce.json
  for k in 0 6 12 24; do
    MC_HOST_MODE=ce MC_CE_CHUNKS=$([ $k = 0 ] || echo $k) python bench.py --config 2 --steps 10 --warmup 3 --ref-seconds 0.1 > gpurun_out/ce.json 2>&1; echo -n "rep$rep ce$k cfg2: "; python scripts/summ.py gpurun_out/ce.json
  done
  python bench.py --config 3 --steps 4 --warmup 3 --ref-seconds 0.1 > gpurun_out/ce.json 2>&1; echo -n "rep$rep default cfg3: "; python scripts/summ.py gpurun_out/ce.json
  for k in 0 32 128; do
    MC_HOST_MODE=ce MC_CE_CHUNKS=$([ $k = 0 ] || echo $k) python bench.py --config 3 --steps 4 --warmup 3 --ref-seconds 0.1 > gpurun_out/ce.json 2>&1; echo -n "rep$rep ce$k cfg3: "; python scripts/summ.py gpurun_out/ce.json
  done
done
