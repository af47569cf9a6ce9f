"""Config-4 product batch with contiguous output rows (ld = n, odd: per-thread
stores in the inverse column pass) vs 16-byte-aligned rows (ld = L: tensor
stores), device time per step (CUDA events, L2 flushed)."""
import os
import sys
import statistics

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01010_b200 as mc  # noqa: E402

p = 2013265921
B, z = 8, 1 << 22
n = 2 * z - 1
g = torch.Generator(device="cuda").manual_seed(4)
a = torch.randint(0, p, (B, z), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
b = torch.randint(0, p, (B, z), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
outs = {"ld=n": torch.empty((B, n), dtype=torch.int32, device="cuda"),
        "ld=L": torch.empty((B, 1 << 23), dtype=torch.int32, device="cuda")[:, :n]}
res = {}
for rep in range(3):
    for name, o in outs.items():
        ts = []
        for i in range(12):
            flush.fill_(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mc.conv_batch(a, b, p, engine="fft_pad", out=o)
            e1.record()
            e1.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        res.setdefault(name, []).append(statistics.median(ts))
assert torch.equal(outs["ld=n"], outs["ld=L"])
for k, v in res.items():
    print(k, " ".join(f"{x:.4f}" for x in v), "ms")
