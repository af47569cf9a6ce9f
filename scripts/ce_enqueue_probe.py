"""Host-mode probe at cfg2 sizes: host enqueue time of one mc_conv_host_async
call, its device time when the GPU is gated (all work enqueued before it
starts), and the ungated end-to-end time, per host mode."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_01010_b200 import _native
lib = _native.lib()
B, z1, z2, p = 4096, 1500, 2100, 2013265921
n = z1 + z2 - 1
a = torch.randint(0, p, (B, z1), dtype=torch.int64).to(torch.int32).pin_memory()
b = torch.randint(0, p, (B, z2), dtype=torch.int64).to(torch.int32).pin_memory()
c = torch.empty((B, n), dtype=torch.int32).pin_memory()
st = torch.cuda.current_stream()
def call():
    _native.check(lib.mc_conv_host_async(1, a.data_ptr(), z1, z1, b.data_ptr(), z2, z2, c.data_ptr(), n, B, p, 0, st.cuda_stream))
for mode in sys.argv[1:]:
    os.environ["MC_HOST_MODE"] = mode if mode != "default" else ""
    call(); torch.cuda.synchronize()
    ref = c.clone()
    host, gated, ungated = [], [], []
    for _ in range(5):
        torch.cuda.synchronize()
        torch.cuda._sleep(10_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        t0 = time.perf_counter(); call(); host.append((time.perf_counter() - t0) * 1e3)
        e1.record(st); torch.cuda.synchronize(); gated.append(e0.elapsed_time(e1))
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); call(); st.synchronize(); e1.record(st); torch.cuda.synchronize()
        ungated.append(e0.elapsed_time(e1))
    assert torch.equal(c, ref)
    print(f"{mode:8s} chunks={os.environ.get('MC_CE_CHUNKS','-')} host enqueue {min(host):.3f} ms  gated device {min(gated):.3f} ms  ungated {min(ungated):.3f} ms (median {sorted(ungated)[2]:.3f})", flush=True)
