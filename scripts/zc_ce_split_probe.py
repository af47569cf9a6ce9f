"""Would splitting a config-2 batch between the zero-copy kernel and the
copy engines use more of the PCIe link?  Gated device times: zero-copy call
on all rows; zero-copy on a fraction f of the rows while the copy engines
move the other rows' operands H2D and products D2H (no kernel for them --
an upper bound for the split)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MC_HOST_MODE"] = "zc"
import torch
from paper_1609_01010_b200 import _native
lib = _native.lib()
B, z1, z2, p = 4096, 1500, 2100, 2013265921
n = z1 + z2 - 1
a = torch.randint(0, p, (B, z1), dtype=torch.int64).to(torch.int32).pin_memory()
b = torch.randint(0, p, (B, z2), dtype=torch.int64).to(torch.int32).pin_memory()
c = torch.empty((B, n), dtype=torch.int32).pin_memory()
da = torch.empty((B, z1), dtype=torch.int32, device="cuda")
db = torch.empty((B, z2), dtype=torch.int32, device="cuda")
dc = torch.zeros((B, n), dtype=torch.int32, device="cuda")
main = torch.cuda.current_stream()
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

def zc(r0, r1, st):
    _native.check(lib.mc_conv_host_async(1, a[r0].data_ptr(), z1, z1, b[r0].data_ptr(), z2, z2,
                                         c[r0].data_ptr(), n, r1 - r0, p, 0, st.cuda_stream))

def gated(f):
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        torch.cuda._sleep(5_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for s in (s1, s2, s3):
            s.wait_stream(main)
        f()
        for s in (s1, s2, s3):
            main.wait_stream(s)
        e1.record(main); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best

print("zero copy, all rows      %.3f ms" % gated(lambda: zc(0, B, s1)), flush=True)
for frac in (0.5, 0.6, 0.7, 0.8):
    k = int(B * frac)
    def f():
        zc(0, k, s1)
        with torch.cuda.stream(s2):
            da[k:].copy_(a[k:], non_blocking=True); db[k:].copy_(b[k:], non_blocking=True)
        with torch.cuda.stream(s3):
            c[k:].copy_(dc[k:], non_blocking=True)
    print("zc %.1f || CE rest        %.3f ms" % (frac, gated(f)), flush=True)
