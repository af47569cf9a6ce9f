"""Split truncated product (tft engine, n = L/2 + m with m <= L/8): a cyclic
L/2-point head on operands folded on load plus a low-product tail that
unwraps the top m coefficients (capi.cu split_tft).  Bit-exact against the C
oracle's conv_tft (reference convolve.py:230-253) over every K where the
split applies, the m boundaries, balanced and lopsided operand lengths,
strided rows (plain loads) and aligned rows (bulk-copy staging), and the
all-(p-1) operands."""

import numpy as np
import pytest
import torch

from conftest import P1, P2, P3

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc
    from paper_1609_01010_b200 import _native
    from gpu_helpers import to_u32_np


def _dev(x, ld=None):
    x = np.ascontiguousarray(x, dtype=np.uint32)
    if ld is None:
        return torch.from_numpy(x.view(np.int32)).cuda()
    buf = torch.zeros((x.shape[0], ld), dtype=torch.int32, device="cuda")
    buf[:, : x.shape[1]] = torch.from_numpy(x.view(np.int32)).cuda()
    return buf[:, : x.shape[1]]


def _rows(K):
    # below K = 10 the split is taken only for batches of >= 2^20 positions
    return 3 if K >= 10 else (1 << 20) >> K


def _check(orc, p, z1, z2, rows, seed, ld=None):
    a = orc.gen_u32(seed, 0, z1, rows, z1, p)
    b = orc.gen_u32(seed, 1, z2, rows, z2, p)
    want, _, _ = orc.conv_batch(a, b, p, orc.ENGINE_TFT)
    ad, bd = _dev(a, ld), _dev(b, ld)
    got = to_u32_np(mc.conv_batch(ad, bd, p, engine="tft"))
    assert np.array_equal(got, want), (p, z1, z2, rows, np.argwhere(got != want)[:4].tolist())
    before = _native.launch_count()  # tables are built now: count one call's kernels
    mc.conv_batch(ad, bd, p, engine="tft")
    return _native.launch_count() - before


@pytest.mark.parametrize("K", list(range(5, 17)))
def test_split_boundaries(orc, K):
    """K <= 14: fused head; K = 15, 16: four-step head (circular L/2-point
    product of the folded operands, plain column loads)."""
    L = 1 << K
    twist = K in (13, 14)  # m in (L/8, L/4]: the twisted quarter piece
    for m in sorted({1, 2, 3, 7, L // 16 - 1, L // 16, L // 16 + 1, L // 8 - 1, L // 8,
                     L // 8 + 1, 3 * L // 16, L // 4 - 1, L // 4}):
        if m < 1 or m > (L // 4 if twist else min(L // 8, 4096)):
            continue
        n = L // 2 + m
        for z1 in sorted({1, 2, (n + 1) // 2, m, L // 2, L // 2 + 1}):
            z2 = n + 1 - z1
            if z1 < 1 or z2 < 1:
                continue
            launches = _check(orc, P3, z1, z2, _rows(K), seed=K * 1000 + m)
            # the head (one fused launch, or three four-step passes) and the
            # tail; up to K = 10 the split is taken for m <= L/16 only
            want = (2 if K <= 14 else 4) if (K > 10 or m <= L // 16) else 1
            assert launches == want, (K, m, z1, launches)


@pytest.mark.parametrize("p", [P1, P2, P3])
def test_split_strided_and_aligned(orc, p):
    for K in (11, 12, 13, 14, 15):
        L = 1 << K
        for m in (5, min(L // 8, 4096)) + ((L // 4,) if K in (13, 14) else ()):
            n = L // 2 + m
            z1 = (n + 1) // 2
            z2 = n + 1 - z1
            _check(orc, p, z1, z2, 4, seed=7 + K, ld=z2 + 5)    # odd stride: plain loads
            _check(orc, p, z1, z2, 4, seed=9 + K, ld=((z2 + 3) // 4) * 4 + 4)  # bulk copies


def test_split_all_p_minus_1(orc):
    for K in (8, 12, 14):
        L = 1 << K
        for m in (1, L // 8) + ((L // 4,) if K == 14 else ()):
            n = L // 2 + m
            z1 = (n + 1) // 2
            z2 = n + 1 - z1
            rows = _rows(K)
            a = np.full((rows, z1), P3 - 1, dtype=np.uint32)
            b = np.full((rows, z2), P3 - 1, dtype=np.uint32)
            want, _, _ = orc.conv_batch(a[:1], b[:1], P3, orc.ENGINE_TFT)
            got = to_u32_np(mc.conv_batch(_dev(a), _dev(b), P3, engine="tft"))
            assert np.array_equal(got, np.repeat(want, rows, axis=0)), (K, m)


def test_split_not_taken_past_quarter(orc):
    """m > L/4 keeps a single launch (the complete transform at fused sizes)
    or the relaxed four-step passes."""
    L = 4096
    n = L // 2 + L // 4 + 1
    z1 = (n + 1) // 2
    assert _check(orc, P2, z1, n + 1 - z1, 3, seed=5) == 1
    L = 1 << 17
    n = L // 2 + 4097  # tail beyond a fused launch
    z1 = (n + 1) // 2
    assert _check(orc, P3, z1, n + 1 - z1, 2, seed=6) == 3


def test_split_poly_mul_counters():
    """poly_mul through the split path: normalized result and the
    reference's analytic TFT counters (convolve.py:230-253)."""
    fp = mc.FourierPrime.from_modulus(P2)
    rng = np.random.default_rng(3)
    a = mc.DensePoly(fp, tuple(int(x) for x in rng.integers(0, P2, 1030)))
    b = mc.DensePoly(fp, tuple(int(x) for x in rng.integers(0, P2, 1031)))
    cnt = mc.OpCounters()
    r = mc.poly_mul(a, b, mc.ConvRequest(fp, engine="tft", counters=cnt))
    r2 = mc.poly_mul(a, b, mc.ConvRequest(fp, engine="fft_pad"))
    assert r == r2 and len(r.coeffs) == 2060
    assert cnt.butterflies > 0


@pytest.mark.parametrize("keep", ["0", "1"])
@pytest.mark.parametrize("K", [7, 10, 12, 13])
def test_truncated_schedule_both_ways(orc, K, keep, monkeypatch):
    """NT = 11..15 of 16 blocks: the tft engine runs the complete transform
    (measured faster), or with MC_TFT_KEEP_NT=1 the relaxed truncated
    kernel (van der Hoeven inverse over the top four levels, Harvey ranges
    for p < 2^30) -- both bit-exact vs the oracle's conv_tft."""
    monkeypatch.setenv("MC_TFT_KEEP_NT", keep)
    L = 1 << K
    G = L // 16
    for p in (P2, P3):
        for nt in range(11, 16):
            n = nt * G - (G // 3 if nt % 2 else 0)
            for z1 in sorted({1, (n + 1) // 2, n - 3}):
                _check(orc, p, z1, n + 1 - z1, 3, seed=K * 100 + nt)
