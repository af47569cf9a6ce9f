# ncu capture of the fused kernel for a given config: bash scripts/gpu_prof.sh <cfg> <tag>
CFG=${1:-2}; TAG=${2:-v}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py --config $CFG --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_small -s 2 -c 1 -o gpurun_out/prof_cfg${CFG}_$TAG python bench.py --config $CFG --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
