# multi-rank bench path on one GPU (gloo for the host-side collectives)
for c in 2 5; do
  BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config $c --steps 3 --warmup 3 \
    --ref-seconds 0.2 > gpurun_out/mr_cfg$c.json 2> gpurun_out/mr_cfg$c.err
  echo "cfg$c rc=$?"; tail -c 600 gpurun_out/mr_cfg$c.json; echo
done
BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --impl reference --steps 2 --warmup 3 \
    --ref-step-seconds 0.2 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo "ref rc=$?"; cat gpurun_out/mr_ref.json | head -c 300
