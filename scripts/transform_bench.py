"""Standalone transforms through the C ABI: device time of
mc_ntt / mc_tft / mc_itft on batches, and the equivalent butterfly rate."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_01010_b200 as mc
from paper_1609_01010_b200 import _native
lib = _native.lib()
st = torch.cuda.current_stream()
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps): fn()
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
out = []
p = 2013265921
for K, B in ((12, 4096), (20, 1), (23, 1)):
    L = 1 << K
    x = torch.randint(0, p, (B, L), dtype=torch.int64).to(torch.int32).cuda()
    y = torch.empty_like(x)
    ms = timeit(lambda: _native.check(lib.mc_ntt(x.data_ptr(), y.data_ptr(), K, B, p, 0, st.cuda_stream)))
    bf = B * (L // 2) * K
    out.append({"op": "moddft", "L": L, "batch": B, "ms": ms, "Gbf_per_s": bf / ms / 1e6})
    n, z = (3599, 2100) if K == 12 else (L - 1, L // 2)
    xz = x[:, :z].contiguous()
    yt = torch.empty((B, n), dtype=torch.int32, device="cuda")
    ms = timeit(lambda: _native.check(lib.mc_tft(xz.data_ptr(), z, yt.data_ptr(), n, K, B, p, st.cuda_stream)))
    bf = B * mc.transform.tft_count(L, z, n)
    out.append({"op": "tft", "L": L, "z": z, "n": n, "batch": B, "ms": ms, "Gbf_per_s": bf / ms / 1e6})
    yi = torch.empty((B, n), dtype=torch.int32, device="cuda")
    ms = timeit(lambda: _native.check(lib.mc_itft(yt.data_ptr(), yi.data_ptr(), n, K, B, p, st.cuda_stream)))
    bf = B * mc.transform.itft_count(L, n)
    out.append({"op": "itft", "L": L, "n": n, "batch": B, "ms": ms, "Gbf_per_s": bf / ms / 1e6})
for o in out:
    print(json.dumps(o))
