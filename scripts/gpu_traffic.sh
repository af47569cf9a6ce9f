# per-step DRAM traffic of our kernels (launch lists with dram metrics) for configs 1, 3, 4, 5
for c in 1 3 4 5; do
  python bench.py --config $c --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/tr_plain$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
      --log-file gpurun_out/traffic_cfg$c.csv python bench.py --config $c --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/tr_ncu$c.log 2>&1
  echo "cfg$c rc=$?"
done
