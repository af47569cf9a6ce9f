# standalone transforms: GPU parity tests + device-time bench (row-resident vs level-scheduled)
timeout 900 python -m pytest tests/test_gpu_transforms.py -x -q 2>&1 | tail -4
python scripts/transform_bench.py > gpurun_out/xf_rows.jsonl 2>&1; cat gpurun_out/xf_rows.jsonl
MC_XFORM_LEVELS=1 python scripts/transform_bench.py > gpurun_out/xf_levels.jsonl 2>&1; cat gpurun_out/xf_levels.jsonl
