"""Small invocations of every shared-memory / async-copy kernel, one scenario
per process, for compute-sanitizer (racecheck / synccheck / memcheck).

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py fused_tma

Each case checks its own output against the C oracle, so a run that the
sanitizer passes is also a correct run.  Scenarios:

  fused_tma     conv_small_kernel, K = 12 / 13, bulk-copy (TMA) row prefetch,
                tft + fft_pad (device-resident operands)
  fused_small   conv_small_kernel, K = 6 / 9 (several products per CTA)
  fused_host    conv_small_kernel reading and writing page-locked host rows
                (zero copy: bulk prefetch in, bulk-store epilogue out)
  fourstep      col_fwd_tma / row_conv / col_inv_async, L = 2^18 (R = 64)
  rowprefetch   the same with the row pass's L2 bulk prefetch forced on
  three_primes  mc_mul_three_primes at a four-step size (crt fused path)
  transforms    xform_small / rows_kernel (moddft / tft / itft)
"""

from __future__ import annotations

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

P1, P2, P3 = 469762049, 998244353, 2013265921


def _conv_case(orc, mc, torch, p, z1, z2, B, engines=("tft", "fft_pad"), host=False):
    a = orc.gen_u32(77, 0, z1, B, z1, p)
    b = orc.gen_u32(77, 1, z2, B, z2, p)
    want, _, _ = orc.conv_batch(a, b, p, threads=8)
    at = torch.from_numpy(a.view(np.int32))
    bt = torch.from_numpy(b.view(np.int32))
    if host:
        at, bt = at.pin_memory(), bt.pin_memory()
    else:
        at, bt = at.cuda(), bt.cuda()
    for eng in engines:
        if host:
            out = torch.empty((B, z1 + z2 - 1), dtype=torch.int32).pin_memory()
            mc.conv_batch(at, bt, p, engine=eng, out=out)
            torch.cuda.synchronize()
            got = out.numpy().view(np.uint32)
        else:
            got = mc.conv_batch(at, bt, p, engine=eng).cpu().numpy().view(np.uint32)
        assert np.array_equal(got, want), (p, z1, z2, eng)


def main(case: str) -> None:
    import torch

    import paper_1609_01010_b200 as mc
    from oracle import oracle as orc

    torch.cuda.set_device(0)
    if case == "fused_tma":
        _conv_case(orc, mc, torch, P3, 1500, 2100, 6)
        _conv_case(orc, mc, torch, P2, 4096, 4096, 3)
    elif case == "fused_small":
        _conv_case(orc, mc, torch, P1, 20, 30, 40)
        _conv_case(orc, mc, torch, P3, 300, 200, 9)
    elif case == "fused_host":
        _conv_case(orc, mc, torch, P3, 1500, 2100, 6, host=True)
    elif case in ("fourstep", "rowprefetch"):
        _conv_case(orc, mc, torch, P3, 1 << 17, (1 << 17) - 5, 1)
        _conv_case(orc, mc, torch, P1, 100000, 90000, 1, engines=("fft_pad",))
    elif case == "three_primes":
        rng = np.random.default_rng(3)
        a = rng.integers(0, 1 << 30, 40000, dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, 1 << 30, 30000, dtype=np.uint64).astype(np.uint32)
        got = mc.mul_three_primes_tensor(torch.from_numpy(a.view(np.int32)).cuda(),
                                         torch.from_numpy(b.view(np.int32)).cuda())
        assert np.array_equal(got.cpu().numpy().view(np.uint32), orc.mul_three_primes(a, b))
    elif case == "transforms":
        fp = mc.FourierPrime.from_modulus(P3)
        for L in (64, 4096, 16384):
            t = mc.get_table(fp, L)
            x = orc.gen_u32(5, 0, L, 1, L, P3)[0].tolist()
            y = mc.moddft(x, t)
            assert mc.moddft(y, t, "inv") == x
            n = L - L // 3
            s = mc.tft(t, x[: n // 2], n)
            u = mc.itft(t, s)
            assert u[: n // 2] == [v * L % P3 for v in x[: n // 2]]
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print("ok", case)


if __name__ == "__main__":
    main(sys.argv[1])
