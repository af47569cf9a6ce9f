"""Device time of four-step products (fft_pad, p3) over K = 17..23 and batches 1, 2, 4:
python scripts/fourstep_sizes.py   (A/B: MC_SMALL_COL_TILES=0|1)"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_01010_b200 as mc

P3 = 2013265921
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for K in range(17, 24):
    for batch in (1, 2, 4):
        z = 1 << (K - 1)
        if 8 * (1 << K) * batch > (1 << 30):
            continue
        g = torch.Generator(device="cuda").manual_seed(K * 7 + batch)
        a = torch.randint(0, P3, (batch, z), dtype=torch.int32, device="cuda", generator=g)
        b = torch.randint(0, P3, (batch, z), dtype=torch.int32, device="cuda", generator=g)
        for _ in range(3):
            mc.conv_batch(a, b, P3, engine="fft_pad")
        ts = []
        for _ in range(10):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mc.conv_batch(a, b, P3, engine="fft_pad")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(f"K={K} batch={batch} median_us={ts[len(ts) // 2]:.1f} min_us={ts[0]:.1f}", flush=True)
