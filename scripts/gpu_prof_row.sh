python bench.py --config 4 --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/plain_row.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:row_conv -s 2 -c 1 -o gpurun_out/prof_cfg4_row python bench.py --config 4 --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/ncu_row.log 2>&1
echo "rc=$?"
