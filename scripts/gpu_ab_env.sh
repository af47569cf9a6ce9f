# alternating A/B of an environment switch on the given configs
# usage: bash scripts/gpu_ab_env.sh "4 5" MC_NO_OUT_TMA=1 [tests...]
CFGS=$1; ENVB=$2; shift 2
[ $# -gt 0 ] && timeout 1500 python -m pytest "$@" -x -q 2>&1 | tail -3
for rep in 1 2; do
  for v in new base; do
    for c in $CFGS; do
      if [ $v = base ]; then env $ENVB python bench.py --config $c --configs head --steps 20 --warmup 5 --ref-seconds 0.1 > gpurun_out/ab.json 2>gpurun_out/ab.err;
      else python bench.py --config $c --configs head --steps 20 --warmup 5 --ref-seconds 0.1 > gpurun_out/ab.json 2>gpurun_out/ab.err; fi
      echo -n "rep$rep $v cfg$c: "; python scripts/summ.py gpurun_out/ab.json
    done
  done
done
