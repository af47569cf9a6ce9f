# host NUMA placement vs the zero-copy host path (cfg2 sizes)
nvidia-smi topo -m 2>&1 | head -12
lscpu | grep -i -E "numa|socket|^cpu\(s\)"
python - <<'PY'
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
try:
    print("gpu0 cpu affinity mask words:", [hex(x) for x in pynvml.nvmlDeviceGetCpuAffinity(h, 4)])
except Exception as e:
    print("affinity query failed", e)
PY
for node in 0 1; do
  if numactl -H >/dev/null 2>&1; then
    echo "== numactl node $node"; numactl --cpunodebind=$node --membind=$node python scripts/ce_enqueue_probe.py zc 2>&1 | tail -1
  fi
done
echo "== default"; python scripts/ce_enqueue_probe.py zc 2>&1 | tail -1
