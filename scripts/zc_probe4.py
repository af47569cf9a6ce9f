"""Copy-engine H2D of the operands alongside a kernel that reads device
memory and writes products to host by bulk stores (cfg2 shapes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_01010_b200 as mc
from paper_1609_01010_b200 import _native
p, B, z1, z2 = 2013265921, 4096, 1500, 2100
n = z1 + z2 - 1
g = torch.Generator().manual_seed(1)
a = torch.randint(0, p, (B, z1), generator=g, dtype=torch.int64).to(torch.int32)
b = torch.randint(0, p, (B, z2), generator=g, dtype=torch.int64).to(torch.int32)
ah, bh = a.pin_memory(), b.pin_memory()
ad, bd = a.cuda(), b.cuda()
ad2, bd2 = torch.empty_like(ad), torch.empty_like(bd)
ch = torch.empty((B, n), dtype=torch.int32).pin_memory()
main = torch.cuda.current_stream()
s2 = torch.cuda.Stream()
def kern():
    _native.check(_native.lib().mc_conv_tft(ad.data_ptr(), z1, z1, bd.data_ptr(), z2, z2, ch.data_ptr(), n, B, p, main.cuda_stream))
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(reps): fn()
    e1.record(main); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d():
    s2.wait_stream(main)
    with torch.cuda.stream(s2):
        ad2.copy_(ah, non_blocking=True); bd2.copy_(bh, non_blocking=True)
    main.wait_stream(s2)
def both():
    s2.wait_stream(main)
    with torch.cuda.stream(s2):
        ad2.copy_(ah, non_blocking=True); bd2.copy_(bh, non_blocking=True)
    kern()
    main.wait_stream(s2)
os.environ["MC_BULK_OUT"] = "1"
print(f"kernel device-in host-out : {timeit(kern):.3f} ms")
print(f"H2D copy engine 59 MB     : {timeit(h2d):.3f} ms")
print(f"both concurrently         : {timeit(both):.3f} ms")
