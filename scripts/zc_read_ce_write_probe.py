"""Can kernel zero-copy READS of the operands run alongside copy-engine D2H
of the products at full PCIe rate?  cfg2 sizes: the fused kernel reading
page-locked host rows (UVA) into a device output, and a 59 MB D2H on a
second stream -- alone and concurrently (device time, CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_01010_b200 import _native
lib = _native.lib()
B, z1, z2, p = 4096, 1500, 2100, 2013265921
n = z1 + z2 - 1
a = torch.randint(0, p, (B, z1), dtype=torch.int64).to(torch.int32).pin_memory()
b = torch.randint(0, p, (B, z2), dtype=torch.int64).to(torch.int32).pin_memory()
ad, bd = a.cuda(), b.cuda()
cd = torch.empty((B, n), dtype=torch.int32, device="cuda")
src = torch.randint(0, p, (B, n), dtype=torch.int64).to(torch.int32).cuda()
dst = torch.empty((B, n), dtype=torch.int32).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()

def kern(x, y, st):
    _native.check(lib.mc_conv_tft(x.data_ptr(), z1, z1, y.data_ptr(), z2, z2, cd.data_ptr(), n, B, p, st.cuda_stream))

def timed(fns):
    torch.cuda.synchronize()
    torch.cuda._sleep(5_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for s, f in fns:
        s.wait_stream(main)
        with torch.cuda.stream(s):
            f(s)
    for s, _ in fns:
        main.wait_stream(s)
    e1.record(main); torch.cuda.synchronize()
    return e0.elapsed_time(e1)

k_dev = lambda s: kern(ad, bd, s)
k_zc = lambda s: kern(a, b, s)
d2h = lambda s: dst.copy_(src, non_blocking=True)
for name, fns in (("kernel, device inputs", [(s1, k_dev)]), ("kernel, zero-copy inputs", [(s1, k_zc)]),
                  ("D2H 59 MB", [(s2, d2h)]), ("zero-copy kernel || D2H", [(s1, k_zc), (s2, d2h)]),
                  ("device kernel || D2H", [(s1, k_dev), (s2, d2h)])):
    t = min(timed(fns) for _ in range(5))
    print(f"{name:28s} {t:.3f} ms", flush=True)
