# A/B prebuilt library variants against the working-tree library, alternated:
# bash scripts/variant_ab.sh "2 3 4" "alu1 alu2"
CFGS=${1:-"2 3"}; VARS=${2:-""}
cp paper_1609_01010_b200/_lib/libmodconv_b200.so /tmp/lib_base.so
for rep in 1 2; do
  for v in base $VARS; do
    if [ $v = base ]; then cp /tmp/lib_base.so paper_1609_01010_b200/_lib/libmodconv_b200.so; else cp variants/lib_$v.so paper_1609_01010_b200/_lib/libmodconv_b200.so; fi
    for c in $CFGS; do
      python bench.py --config $c --configs head --steps 20 --warmup 5 --ref-seconds 0.1 > gpurun_out/ab.json 2>&1
      echo -n "rep$rep $v cfg$c: "; python scripts/summ.py gpurun_out/ab.json
    done
  done
done
cp /tmp/lib_base.so paper_1609_01010_b200/_lib/libmodconv_b200.so
