# parity of the lazy-range kernels + A/B against MC_NO_LAZY=1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for v in "" 1; do
  echo "== MC_NO_LAZY=$v"
  for c in 3 5 1 2; do
    st=20; [ $c -ge 4 ] && st=10
    MC_NO_LAZY=$v python bench.py --config $c --steps $st --warmup 4 --ref-seconds 0.1 > gpurun_out/lz$c.json 2>&1; python scripts/summ.py gpurun_out/lz$c.json
  done
done
