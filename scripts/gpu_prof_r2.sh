# round-2 captures: ncu --set full of the four-step passes (config 4: col_fwd_tma, row_conv,
# col_inv_async; config 5: col_inv3_crt) and the fused kernel (config 2); then the
# multi-rank bench plumbing (2 ranks sharing the one GPU, gloo host collectives)
mkdir -p gpurun_out/r2
B="python bench.py --configs head --steps 2 --warmup 3 --ref-seconds 0.1"
$B --config 4 > /dev/null 2>&1 || echo "plain cfg4 failed"
for k in col_fwd_tma row_conv col_inv_async; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/r2/prof_cfg4_$k $B --config 4 > gpurun_out/r2/ncu_cfg4_$k.log 2>&1; echo "cfg4 $k rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:col_inv3 -s 1 -c 1 -o gpurun_out/r2/prof_cfg5_col_inv3 $B --config 5 > gpurun_out/r2/ncu_cfg5.log 2>&1; echo "cfg5 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:conv_small -s 2 -c 1 -o gpurun_out/r2/prof_cfg2 $B --config 2 > gpurun_out/r2/ncu_cfg2.log 2>&1; echo "cfg2 rc=$?"
BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --configs 2,5,4 --steps 5 --warmup 3 --ref-seconds 0.1 > gpurun_out/r2/multirank_gloo_shared_gpu.json 2> gpurun_out/r2/multirank.err; echo "multirank rc=$?"; tail -3 gpurun_out/r2/multirank.err
