# round-2 final evidence at HEAD: gpu_prof_r2b.sh's captures plus the config-5
# forward column and row passes and the config-3 kernel
bash scripts/gpu_prof_r2b.sh
B="python bench.py --configs head --steps 2 --warmup 3 --ref-seconds 0.1"
F="ncu --set full --clock-control none --import-source on"
$F -k regex:conv_small -s 2 -c 1 -o gpurun_out/r2prof/prof_cfg3 $B --config 3 > /dev/null 2>&1; echo "cfg3 full rc=$?"
for k in col_fwd_tma row_conv; do
  $F -k regex:$k -s 3 -c 1 -o gpurun_out/r2prof/prof_cfg5_$k $B --config 5 > /dev/null 2>&1; echo "cfg5 $k rc=$?"
done
# gpurun copies back at most 64 MiB: keep the text summaries, drop the reports
for r in gpurun_out/r2prof/*.ncu-rep; do
  python scripts/ncu_summary.py $r > ${r%.ncu-rep}_summary.txt 2>&1
done
python scripts/ncu_segments.py gpurun_out/r2prof/prof_cfg2.ncu-rep > gpurun_out/r2prof/prof_cfg2_segments.txt 2>&1
python scripts/ncu_segments.py gpurun_out/r2prof/prof_cfg3.ncu-rep > gpurun_out/r2prof/prof_cfg3_segments.txt 2>&1
rm -f gpurun_out/r2prof/*.ncu-rep
du -sh gpurun_out
