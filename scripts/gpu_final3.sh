# round-end evidence at HEAD: bench lines (all configs + reference arm), cfg2 launch list,
# ncu --set full of the cfg2 kernel, cfg3 kernel capture
python bench.py > gpurun_out/f3_cfg2.json 2> gpurun_out/f3_cfg2.err; python scripts/summ.py gpurun_out/f3_cfg2.json
for c in 1 3 4 5; do python bench.py --config $c > gpurun_out/f3_cfg$c.json 2> gpurun_out/f3_cfg$c.err; python scripts/summ.py gpurun_out/f3_cfg$c.json; done
python bench.py --impl reference > gpurun_out/f3_ref.json 2>&1; head -c 200 gpurun_out/f3_ref.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg2_final.csv \
  python bench.py --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/f3_ncu1.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:conv_small -s 2 -c 1 -o gpurun_out/prof_cfg2_final2 \
  python bench.py --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/f3_ncu2.log 2>&1; echo "full rc=$?"
ncu --set full --clock-control none -k regex:conv_small -s 2 -c 1 -o gpurun_out/prof_cfg3_final \
  python bench.py --config 3 --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/f3_ncu3.log 2>&1; echo "full3 rc=$?"
