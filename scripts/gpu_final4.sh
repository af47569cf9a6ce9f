# bench lines at HEAD (all configs, reference arm) with per-step times
for c in 2 1 3 4 5; do BENCH_STEP_TIMES=1 python bench.py --config $c > gpurun_out/f4_cfg$c.json 2> gpurun_out/f4_cfg$c.err; python scripts/summ.py gpurun_out/f4_cfg$c.json; grep step gpurun_out/f4_cfg$c.err | cut -c1-160; done
python bench.py --impl reference > gpurun_out/f4_ref.json 2>&1; head -c 150 gpurun_out/f4_ref.json; echo
