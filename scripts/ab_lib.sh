# A/B: the working-tree library (new) vs variants/lib_head.so (old), alternated twice
# usage: bash scripts/ab_lib.sh "2 3 4"
CFGS=${1:-"2 3"}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
cp paper_1609_01010_b200/_lib/libmodconv_b200.so /tmp/lib_new.so
for rep in 1 2; do
  for v in new head; do
    if [ $v = new ]; then cp /tmp/lib_new.so paper_1609_01010_b200/_lib/libmodconv_b200.so; else cp variants/lib_head.so paper_1609_01010_b200/_lib/libmodconv_b200.so; fi
    for c in $CFGS; do
      python bench.py --config $c --configs head --steps 20 --warmup 5 --ref-seconds 0.1 > gpurun_out/ab.json 2>&1
      echo -n "rep$rep $v cfg$c: "; python scripts/summ.py gpurun_out/ab.json
    done
  done
done
cp /tmp/lib_new.so paper_1609_01010_b200/_lib/libmodconv_b200.so
