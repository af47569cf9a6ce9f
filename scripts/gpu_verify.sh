# verify HEAD on the box: GPU tests, smoke, default bench + all configs
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/v_default.json 2> gpurun_out/v_default.err; python scripts/summ.py gpurun_out/v_default.json
for c in 1 3 4 5; do python bench.py --config $c --ref-seconds 1 > gpurun_out/v_cfg$c.json 2> gpurun_out/v_cfg$c.err; python scripts/summ.py gpurun_out/v_cfg$c.json; done
python bench.py --impl reference > gpurun_out/v_ref.json 2>&1; head -c 600 gpurun_out/v_ref.json
