python scripts/ubench.py > gpurun_out/ubench_r02.json 2>&1; cat gpurun_out/ubench_r02.json
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/gputests.txt
cat gpurun_out/gputests.txt
