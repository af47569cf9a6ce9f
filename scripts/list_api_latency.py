"""Latency of the call-compatible list API (one product per call), the way a
reference user calls it: poly_mul / lin_conv_fft_pad / conv_tft on Python lists."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import random
import torch
import paper_1609_01010_b200 as mc
for p, z1, z2, eng in ((469762049, 1024, 1024, "fft_pad"), (2013265921, 1500, 2100, "tft"),
                        (998244353, 4096, 4096, "fft_pad")):
    fp = mc.FourierPrime.from_modulus(p)
    rnd = random.Random(1)
    u = [rnd.randrange(p) for _ in range(z1)]
    v = [rnd.randrange(p) for _ in range(z2)]
    req = mc.ConvRequest(fp, engine=eng)
    a, b = mc.DensePoly(fp, tuple(u)), mc.DensePoly(fp, tuple(v))
    fn = mc.lin_conv_fft_pad if eng == "fft_pad" else mc.conv_tft
    for name, call in (("poly_mul", lambda: mc.poly_mul(a, b, req)), (fn.__name__, lambda: fn(u, v, req))):
        for _ in range(3): call()
        ts = []
        for _ in range(30):
            t0 = time.perf_counter(); call(); ts.append(time.perf_counter() - t0)
        print(f"{name:18s} p={p} {z1}x{z2} {eng:8s} median {1e3 * statistics.median(ts):.3f} ms")
