# round-2 evidence at HEAD: per-launch lists with DRAM bytes for every config,
# ncu --set full of the headline kernel (config 2), the three four-step passes
# (config 4) and the fused inverse + CRT pass (config 5)
mkdir -p gpurun_out/r2prof
B="python bench.py --configs head --steps 2 --warmup 3 --ref-seconds 0.1"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for c in 1 2 3 4 5; do
  $B --config $c > /dev/null 2>&1 && ncu --metrics $M --clock-control none -c 60 --csv --log-file gpurun_out/r2prof/launches_cfg$c.csv $B --config $c > /dev/null 2>&1
  echo "cfg$c launches rc=$?"
done
F="ncu --set full --clock-control none --import-source on"
$F -k regex:conv_small -s 2 -c 1 -o gpurun_out/r2prof/prof_cfg2 $B --config 2 > /dev/null 2>&1; echo "cfg2 full rc=$?"
for k in col_fwd_tma row_conv col_inv_async; do
  $F -k regex:$k -s 1 -c 1 -o gpurun_out/r2prof/prof_cfg4_$k $B --config 4 > /dev/null 2>&1; echo "cfg4 $k rc=$?"
done
$F -k regex:col_inv3 -s 1 -c 1 -o gpurun_out/r2prof/prof_cfg5_inv3 $B --config 5 > /dev/null 2>&1; echo "cfg5 inv3 rc=$?"
