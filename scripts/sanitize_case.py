"""Small invocations of every kernel family for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_01010_b200 as mc
from oracle import oracle
P3, P2 = 2013265921, 998244353
def conv(z1, z2, B, p, eng):
    a = oracle.gen_u32(1, 0, 0, B, z1, p); b = oracle.gen_u32(1, 1, 0, B, z2, p)
    got = mc.conv_batch(torch.from_numpy(a.view(np.int32)).cuda(), torch.from_numpy(b.view(np.int32)).cuda(), p, engine=eng)
    want, _, _ = oracle.conv_batch(a, b, p)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want), (z1, z2, eng)
conv(1500, 2100, 4, P3, "tft")      # K=12 fused, NT=15, TMA prefetch
conv(4096, 4096, 2, P2, "fft_pad")  # K=13 fused
conv(700, 300, 3, P2, "tft")        # K=10, several products per CTA
conv(5, 3, 3, P2, "tft")            # tiny
conv(9000, 9000, 1, P3, "tft")      # K=15 four-step, truncated
fp = mc.FourierPrime.from_modulus(P3)
t = mc.get_table(fp, 64)
x = list(range(1, 40))
assert mc.itft(t, mc.tft(t, x, 50)) == [v * 64 % P3 for v in x] + [0] * 11
print(mc.mul_three_primes([3, 5, 7], [11, 13]))
print("sanitize case ok")
