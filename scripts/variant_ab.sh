# A/B prebuilt library variants: bash scripts/variant_ab.sh "2 3 4" [test]
CFGS=${1:-"2 3"}; TEST=${2:-}
cp paper_1609_01010_b200/_lib/libmodconv_b200.so /tmp/lib_base.so
for f in /tmp/lib_base.so variants/lib_*.so; do
  cp $f paper_1609_01010_b200/_lib/libmodconv_b200.so
  echo "== $f"
  if [ -n "$TEST" ]; then timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_fourstep.py tests/test_gpu_split.py -q -x 2>&1 | tail -1; fi
  for c in $CFGS; do
    st=20; [ $c -ge 4 ] && st=10
    python bench.py --config $c --steps $st --warmup 4 --ref-seconds 0.1 > gpurun_out/ab$c.json 2>&1 && python scripts/summ.py gpurun_out/ab$c.json
  done
done
cp /tmp/lib_base.so paper_1609_01010_b200/_lib/libmodconv_b200.so
