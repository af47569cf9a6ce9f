"""Can SM-initiated host reads (the kernel's bulk prefetch) and copy-engine
D2H writes share PCIe at full rate?  cfg2 shapes."""
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
ch = torch.empty((B, n), dtype=torch.int32).pin_memory()
cd = torch.empty((B, n), dtype=torch.int32, device="cuda")
cd2 = torch.randint(0, p, (B, n), dtype=torch.int32, device="cuda")
main = torch.cuda.current_stream()
s2 = torch.cuda.Stream()
def kern(C):
    _native.check(_native.lib().mc_conv_tft(ah.data_ptr(), z1, z1, bh.data_ptr(), z2, z2, C.data_ptr(), n, B, p, main.cuda_stream))
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(reps): fn()
    e1.record(main); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def d2h():
    s2.wait_stream(main)
    with torch.cuda.stream(s2):
        ch.copy_(cd2, non_blocking=True)
    main.wait_stream(s2)
def both():
    s2.wait_stream(main)
    with torch.cuda.stream(s2):
        ch.copy_(cd2, non_blocking=True)
    kern(cd)
    main.wait_stream(s2)
print(f"kernel host-in device-out : {timeit(lambda: kern(cd)):.3f} ms")
print(f"D2H copy engine 59 MB     : {timeit(d2h):.3f} ms")
print(f"both concurrently         : {timeit(both):.3f} ms")
print(f"kernel host-in host-out   : {timeit(lambda: kern(ch)):.3f} ms")
