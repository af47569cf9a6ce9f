cp paper_1609_01010_b200/_lib/libmodconv_b200.so /tmp/lib_base.so
timeout 600 python -m pytest tests/test_gpu_fourstep.py -q -x 2>&1 | tail -1
for f in /tmp/lib_base.so variants/lib_*.so; do
  cp $f paper_1609_01010_b200/_lib/libmodconv_b200.so
  echo "== $f"
  python bench.py --config 4 --steps 10 --warmup 3 --ref-seconds 0.1 > gpurun_out/v4.json 2>&1 && python scripts/summ.py gpurun_out/v4.json
  python bench.py --config 5 --steps 10 --warmup 3 --ref-seconds 0.1 > gpurun_out/v5.json 2>&1 && python scripts/summ.py gpurun_out/v5.json
done
cp /tmp/lib_base.so paper_1609_01010_b200/_lib/libmodconv_b200.so
