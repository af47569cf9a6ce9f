# full measurement pass: tests, all configs, launch list + ncu of the cfg2 kernel
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 1 2 3 4 5; do python bench.py --config $c > gpurun_out/final_cfg$c.json 2> gpurun_out/final_cfg$c.err; python scripts/summ.py gpurun_out/final_cfg$c.json; done
python bench.py --impl reference > gpurun_out/final_ref.json 2>&1; head -c 400 gpurun_out/final_ref.json; echo
python scripts/ubench.py > gpurun_out/ubench.json 2>&1
python bench.py --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/fplain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/final_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/fncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_small -s 2 -c 1 -o gpurun_out/prof_cfg2_final python bench.py --steps 2 --warmup 3 --ref-seconds 0.1 > gpurun_out/fncu2.log 2>&1
echo "ncu rc=$?"
