"""Zero-copy directions in isolation: host-in/device-out, device-in/host-out,
host both ways (kernel launched on raw pointers through the C ABI)."""
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
ch = torch.empty((B, n), dtype=torch.int32).pin_memory()
cd = torch.empty((B, n), dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
def run(A, Bm, C):
    _native.check(_native.lib().mc_conv_tft(A.data_ptr(), z1, z1, Bm.data_ptr(), z2, z2, C.data_ptr(), n, B, p, st.cuda_stream))
def t(A, Bm, C, name):
    run(A, Bm, C); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10): run(A, Bm, C)
    e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:28s} {ms:.3f} ms  in {4*B*(z1+z2)/ms/1e6:.1f} GB/s  out {4*B*n/ms/1e6:.1f} GB/s", flush=True)
t(ad, bd, cd, "device in, device out")
t(ah, bh, cd, "host in, device out")
t(ad, bd, ch, "device in, host out")
t(ah, bh, ch, "host in, host out")
