# four-step change check: four-step/CRT GPU tests, then cfg4/cfg5 with and without the twist tables
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_transforms.py -x -q 2>&1 | tail -3
for c in 4 5; do
  for v in "" 1; do
    MC_NO_TWIST_TABLE=$v python bench.py --config $c --steps 10 --warmup 3 --ref-seconds 0.1 > gpurun_out/fs_${c}_$v.json 2>&1
    echo "cfg$c no_twist_table=$v"; python scripts/summ.py gpurun_out/fs_${c}_$v.json
  done
done
