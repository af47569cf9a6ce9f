# three-primes fused CRT path: parity, then A/B against the per-prime path (MC_NO_FUSED_CRT=1)
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_p2p.py -q -x 2>&1 | tail -3
for rep in 1 2; do
  for v in fused split; do
    env=""; [ $v = split ] && env="MC_NO_FUSED_CRT=1"
    env $env python bench.py --config 5 --configs head --steps 20 --ref-seconds 0.1 > gpurun_out/ab5_$v.json 2>gpurun_out/ab5_$v.err
    python -c "
import json; d=json.load(open('gpurun_out/ab5_$v.json'))
print('$v rep$rep', round(d['ms_per_step']*1e3,1), 'us', d['clocks']['sm_mhz'], 'launches', d['gpu_launches'], 'e2e', round(d['e2e']['value']))"
  done
done
