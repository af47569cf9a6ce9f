# round-end pass at HEAD: GPU tests, smoke, every config, reference arm, transforms, multirank
timeout 1300 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/f2_cfg2.json 2> gpurun_out/f2_cfg2.err; python scripts/summ.py gpurun_out/f2_cfg2.json
for c in 1 3 4 5; do python bench.py --config $c > gpurun_out/f2_cfg$c.json 2> gpurun_out/f2_cfg$c.err; python scripts/summ.py gpurun_out/f2_cfg$c.json; done
python bench.py --impl reference > gpurun_out/f2_ref.json 2>&1; head -c 300 gpurun_out/f2_ref.json; echo
python scripts/transform_bench.py > gpurun_out/f2_xf.jsonl 2>&1; cat gpurun_out/f2_xf.jsonl
