"""Config 2's shape (4096 x (1500 x 2100) mod p3) through both engines:
device time per batch (CUDA events, L2 flushed), alternating, medians."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_01010_b200 as mc  # noqa: E402

p = 2013265921
z1, z2 = int(os.environ.get("Z1", 1500)), int(os.environ.get("Z2", 2100))
g = torch.Generator(device="cuda").manual_seed(2)
a = torch.randint(0, p, (4096, z1), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
b = torch.randint(0, p, (4096, z2), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {e: mc.conv_batch(a, b, p, engine=e) for e in ("tft", "fft_pad")}
assert torch.equal(out["tft"], out["fft_pad"])
res = {e: [] for e in out}
for rep in range(4):
    for e in out:
        ts = []
        for i in range(12):
            flush.fill_(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mc.conv_batch(a, b, p, engine=e, out=out[e])
            e1.record()
            e1.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1) * 1e3)
        res[e].append(statistics.median(ts))
for e, v in res.items():
    print(e, " ".join(f"{x:.1f}" for x in v), "us")
