# A/B the fused kernel across prebuilt library variants (variants/lib_*.so)
cp paper_1609_01010_b200/_lib/libmodconv_b200.so /tmp/lib_base.so
for f in /tmp/lib_base.so variants/lib_*.so; do
  cp $f paper_1609_01010_b200/_lib/libmodconv_b200.so
  echo "== $f"
  python bench.py --steps 30 --warmup 5 --ref-seconds 0.2 > gpurun_out/vb.json 2>&1 && python scripts/summ.py gpurun_out/vb.json
  python bench.py --config 3 --steps 5 --warmup 3 --ref-seconds 0.2 > gpurun_out/vb3.json 2>&1 && python scripts/summ.py gpurun_out/vb3.json
done
cp /tmp/lib_base.so paper_1609_01010_b200/_lib/libmodconv_b200.so
