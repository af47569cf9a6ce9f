timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for mb in 64 128 256 512; do
  echo "== scratch $mb MiB"; MC_FOURSTEP_SCRATCH_MB=$mb python bench.py --config 4 --steps 10 --warmup 3 --ref-seconds 0.2 > gpurun_out/c4.json 2>&1 && python scripts/summ.py gpurun_out/c4.json
done
