# pass-bench variants + per-pipe utilization of each (ncu)
python scripts/ubench.py > gpurun_out/ubench.json 2> gpurun_out/ubench.err && cat gpurun_out/ubench.json && \
ncu --set full --clock-control none -k regex:"pass_bench|ubench_kernel" -c 20 -o gpurun_out/prof_ubench python scripts/ubench.py > gpurun_out/ncu_ub.log 2>&1
echo "rc=$?"
