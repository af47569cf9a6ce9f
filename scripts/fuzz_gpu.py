"""Randomised GPU-vs-oracle parity sweep (a soak beyond the fixed test
cases): random primes (incl. small-adicity ones), engines, operand lengths up
to 2^17 products, batch sizes 1..300, strided rows, pinned-host and device
tensors, standalone transforms and the definition engine, for a time budget.

    python scripts/fuzz_gpu.py [seconds] [seed]

Prints one line per failure and a summary; exit code 1 on any mismatch.
"""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1609_01010_b200 as mc  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1609_01010_b200 import _native  # noqa: E402

PRIMES = [257, 65537, 7340033, 469762049, 998244353, 2013265921, 167772161, 754974721]


def check_conv(rng, stats):
    p = rng.choice(PRIMES)
    fp = mc.FourierPrime.from_modulus(p)
    maxlog = min(fp.two_adicity, 17)
    n = rng.randint(1, 1 << maxlog)
    if rng.random() < 0.25 and maxlog >= 6:  # just past a power of two: split truncated product
        k = rng.randint(5, maxlog - 1)
        n = (1 << k) + rng.randint(1, max(1, (1 << k) // 4))
    z1 = rng.randint(1, n)
    z2 = n + 1 - z1
    L = 1 << (n - 1).bit_length() if n > 1 else 1
    budget = max(1, (1 << 19) // max(L, 1))
    B = rng.randint(1, min(300, budget))
    engine = rng.choice(["tft", "fft_pad", "definition"] if z1 * z2 <= 1 << 20 else ["tft", "fft_pad"])
    a = orc.gen_u32(rng.randrange(1 << 30), 0, 0, B, z1, p)
    b = orc.gen_u32(rng.randrange(1 << 30), 1, 0, B, z2, p)
    if rng.random() < 0.2:
        a[0, :] = p - 1
        b[0, :] = p - 1
    want, _, _ = orc.conv_batch(a, b, p, orc.ENGINE_FFT_PAD, threads=8)
    pad = rng.choice([0, 0, 1, 3, 8])
    at = torch.zeros((B, z1 + pad), dtype=torch.int32)
    bt = torch.zeros((B, z2 + pad), dtype=torch.int32)
    at[:, :z1] = torch.from_numpy(a.view(np.int32))
    bt[:, :z2] = torch.from_numpy(b.view(np.int32))
    where = rng.choice(["cuda", "pinned", "cpu"]) if engine != "definition" else "cuda"
    if where == "cuda":
        at, bt = at.cuda(), bt.cuda()
    elif where == "pinned":
        at, bt = at.pin_memory(), bt.pin_memory()
    got = mc.conv_batch(at[:, :z1], bt[:, :z2], p, engine=engine)
    got = got.cpu().numpy().view(np.uint32)
    ok = np.array_equal(got, want)
    stats["conv"] += 1
    if not ok:
        bad = np.argwhere(got != want)[:3].tolist()
        print(f"FAIL conv p={p} z1={z1} z2={z2} B={B} engine={engine} where={where} pad={pad} "
              f"at {bad}", flush=True)
    return ok


def check_transforms(rng, stats):
    p = rng.choice(PRIMES)
    fp = mc.FourierPrime.from_modulus(p)
    lg = rng.randint(0, min(fp.two_adicity, 16))
    L = 1 << lg
    n = rng.randint(1, L)
    z = rng.randint(1, n)
    B = rng.randint(1, max(1, min(64, (1 << 18) // L)))
    x = orc.gen_u32(rng.randrange(1 << 30), 0, 0, B, z, p)
    sh = torch.cuda.current_stream().cuda_stream
    xt = torch.from_numpy(x.view(np.int32)).cuda()
    y = torch.empty((B, n), dtype=torch.int32, device="cuda")
    _native.check(_native.lib().mc_tft(xt.data_ptr(), z, y.data_ptr(), n, lg, B, p, sh))
    spec = y.cpu().numpy().view(np.uint32)
    back = torch.empty((B, n), dtype=torch.int32, device="cuda")
    _native.check(_native.lib().mc_itft(y.data_ptr(), back.data_ptr(), n, lg, B, p, sh))
    back = back.cpu().numpy().view(np.uint32)
    ok = True
    for r in (0, B - 1):
        ok &= np.array_equal(spec[r], orc.tft(x[r], n, L, p)[0])
        ok &= np.array_equal(back[r], orc.itft(spec[r], L, p)[0])
        xr = np.zeros(n, dtype=np.uint64)
        xr[:z] = x[r]
        ok &= np.array_equal(back[r].astype(np.uint64), xr * L % p)
    stats["xform"] += 1
    if not ok:
        print(f"FAIL transforms p={p} L={L} n={n} z={z} B={B}", flush=True)
    return ok


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = random.Random(seed)
    stats = {"conv": 0, "xform": 0}
    fails = 0
    t0 = time.time()
    while time.time() - t0 < budget:
        ok = check_conv(rng, stats) if rng.random() < 0.7 else check_transforms(rng, stats)
        fails += not ok
    print(f"fuzz: {stats['conv']} batched products, {stats['xform']} transform cases, "
          f"{fails} failures in {time.time() - t0:.0f} s (seed {seed})", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
