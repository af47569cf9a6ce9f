# Race-stress build (compute-sanitizer is closed on this pool): every CTA
# barrier, mbarrier wait and shared-memory exchange is followed / preceded by
# a random sleep of 1/8 of the threads (tma.cuh mc_perturb), then the whole GPU
# parity suite and a randomised soak must stay bit-exact.  A self-test build
# with one exchange barrier removed (-DMC_RACE_SELFTEST) must fail.
mkdir -p gpurun_out/race
MC_EXTRA_FLAGS="-DMC_RACE_CHECK" python -m paper_1609_01010_b200.build > gpurun_out/race/build.log 2>&1 || echo "build failed"
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/race/tests.log 2>&1
echo "race-stress tests rc=$?"; tail -3 gpurun_out/race/tests.log
timeout 600 python scripts/fuzz_gpu.py 300 7 > gpurun_out/race/fuzz.log 2>&1
echo "race-stress fuzz rc=$?"; tail -3 gpurun_out/race/fuzz.log
MC_EXTRA_FLAGS="-DMC_RACE_CHECK -DMC_RACE_SELFTEST" python -m paper_1609_01010_b200.build > gpurun_out/race/build_self.log 2>&1 || echo "selftest build failed"
timeout 900 python -m pytest tests/test_gpu_conv.py -q -p no:cacheprovider > gpurun_out/race/selftest.log 2>&1
echo "selftest (one barrier removed) rc=$? -- expected nonzero"; tail -3 gpurun_out/race/selftest.log
python -m paper_1609_01010_b200.build > /dev/null 2>&1
