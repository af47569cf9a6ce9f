"""GPU parity of the standalone transforms (moddft / tft / itft, reference
transform.py:167-196, :379-529) against the reference's golden vectors and
the C oracle, including the reference's own property sweeps."""

import numpy as np
import pytest
import torch

from conftest import P1, P2, P3

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc
    from paper_1609_01010_b200 import _native, _tensors


def _tab(p, L):
    return mc.get_table(mc.FourierPrime.from_modulus(p), L)


def test_golden_transforms(golden_small):
    for c in golden_small["transforms"]:
        p, L = c["p"], c["L"]
        t = _tab(p, L)
        if c["kind"] == "moddft":
            cnt = mc.OpCounters()
            assert mc.moddft(c["x"], t, "fwd", cnt) == c["fwd"], (p, L)
            assert cnt.butterflies == c["butterflies"]
            assert mc.moddft(c["x"], t, "inv") == c["inv"], (p, L)
        else:
            cnt = mc.OpCounters()
            assert mc.tft(t, c["x"], c["n"], cnt) == c["y"], (p, L, c["n"], len(c["x"]))
            assert cnt.butterflies == c["butterflies"]
            cnt = mc.OpCounters()
            assert mc.itft(t, c["itft_in"], cnt) == c["itft_out"], (p, L, c["n"])
            assert cnt.butterflies == c["itft_butterflies"]


def test_p5_kats(golden_small):
    t = _tab(5, 4)
    for c in golden_small["kats"]["dft_p5"]:
        assert mc.moddft(c["x"], t) == c["y"]
    assert mc.tft(_tab(17, 4), [9], 1) == [9]


def _batched(fn_name, *args):
    return getattr(_native.lib(), fn_name)(*args)


def test_tft_lattice_vs_oracle(orc):
    """Exhaustive (n, z) lattice for L <= 16, sampled z above
    (reference tests/test_transform.py:210-219), batched 3 rows per call."""
    p = P2
    for L in (2, 4, 8, 16, 32, 64, 128):
        lg = L.bit_length() - 1
        for n in range(1, L + 1):
            zs = range(1, n + 1) if L <= 16 else sorted({1, n, max(1, n // 2)})
            for z in zs:
                x = orc.gen_u32(60, 0, L * 1000 + n * 10 + z, 3, z, p)
                want = np.stack([orc.tft(x[r], n, L, p)[0] for r in range(3)])
                xt = torch.from_numpy(x.view(np.int32)).cuda()
                y = torch.empty((3, n), dtype=torch.int32, device="cuda")
                _native.check(_native.lib().mc_tft(xt.data_ptr(), z, y.data_ptr(), n, lg, 3, p,
                                                    _tensors.stream_handle()))
                assert np.array_equal(y.cpu().numpy().view(np.uint32), want), (L, n, z)


@pytest.mark.parametrize("p", [P1, P3])
def test_itft_tft_roundtrip_all_n(orc, p):
    """itft(tft(x)) == L*x for every 1 <= n <= L <= 1024, the reference's
    own range (tests/test_acceptance.py:62-82)."""
    for lg in range(0, 11):
        L = 1 << lg
        for n in range(1, L + 1):
            x = orc.gen_u32(61, 0, L * 1000 + n, 2, n, p)
            xt = torch.from_numpy(x.view(np.int32)).cuda()
            spec = torch.empty((2, n), dtype=torch.int32, device="cuda")
            back = torch.empty((2, n), dtype=torch.int32, device="cuda")
            sh = _tensors.stream_handle()
            _native.check(_native.lib().mc_tft(xt.data_ptr(), n, spec.data_ptr(), n, lg, 2, p, sh))
            _native.check(_native.lib().mc_itft(spec.data_ptr(), back.data_ptr(), n, lg, 2, p, sh))
            got = back.cpu().numpy().view(np.uint32).astype(np.uint64)
            assert np.array_equal(got, x.astype(np.uint64) * L % p), (L, n)
            want_spec = np.stack([orc.tft(x[r], n, L, p)[0] for r in range(2)])
            assert np.array_equal(spec.cpu().numpy().view(np.uint32), want_spec), (L, n)


@pytest.mark.parametrize("lg", [12, 16, 20])
def test_large_transforms_vs_oracle(orc, lg):
    p = P3
    L = 1 << lg
    x = orc.gen_u32(62, 0, lg, 1, L, p)[0]
    t = _tab(p, L)
    fwd = mc.moddft(x.tolist(), t)
    want, _ = orc.moddft(x, p)
    assert fwd == want.tolist()
    assert mc.moddft(fwd, t, "inv") == x.tolist()
    n = L - L // 3
    z = n // 2
    y = mc.tft(t, x[:z].tolist(), n)
    assert y == orc.tft(x[:z], n, L, p)[0].tolist()
    back = mc.itft(t, y)
    assert back == orc.itft(np.array(y, dtype=np.uint32), L, p)[0].tolist()


@pytest.mark.parametrize("lg", list(range(4, 14)))
@pytest.mark.parametrize("p", [P1, P3])
def test_fused_transforms_every_size(orc, lg, p):
    """The fused single-CTA transforms (L = 16 .. 8192): batched moddft both
    ways and tft at several (n, z) against the oracle, all-(p-1) rows
    included."""
    L = 1 << lg
    B = 5
    x = orc.gen_u32(63, 0, lg, B, L, p)
    x[2, :] = p - 1
    sh = _tensors.stream_handle()
    xt = torch.from_numpy(x.view(np.int32)).cuda()
    y = torch.empty_like(xt)
    _native.check(_native.lib().mc_ntt(xt.data_ptr(), y.data_ptr(), lg, B, p, 0, sh))
    fwd = y.cpu().numpy().view(np.uint32)
    for r in (0, 2, 4):
        assert np.array_equal(fwd[r], orc.moddft(x[r], p)[0]), (L, r)
    back = torch.empty_like(xt)
    _native.check(_native.lib().mc_ntt(y.data_ptr(), back.data_ptr(), lg, B, p, 1, sh))
    assert np.array_equal(back.cpu().numpy().view(np.uint32), x)
    for n in sorted({L // 2 + 1, L - L // 5, L - 1, L}):
        for z in sorted({1, n // 3 + 1, n}):
            xz = torch.from_numpy(np.ascontiguousarray(x[:, :z]).view(np.int32)).cuda()
            t = torch.empty((B, n), dtype=torch.int32, device="cuda")
            _native.check(_native.lib().mc_tft(xz.data_ptr(), z, t.data_ptr(), n, lg, B, p, sh))
            got = t.cpu().numpy().view(np.uint32)
            for r in (1, 2):
                assert np.array_equal(got[r], orc.tft(x[r, :z], n, L, p)[0]), (L, n, z, r)


def test_usage_errors():
    t = _tab(257, 8)
    with pytest.raises(ValueError):
        mc.moddft([1, 2, 3], t)
    with pytest.raises(ValueError):
        mc.moddft([1] * 8, t, "sideways")
    with pytest.raises(ValueError):
        mc.tft(t, [1] * 5, 3)
    with pytest.raises(ValueError):
        mc.tft(t, [1] * 5, 9)
    with pytest.raises(ValueError):
        mc.tft(t, [], 1)
    with pytest.raises(ValueError):
        mc.itft(t, [1] * 9)
    with pytest.raises(ValueError):
        mc.itft(t, [])


@pytest.mark.parametrize("lg", [5, 11, 12, 13, 14])
@pytest.mark.parametrize("p", [P1, P3])
def test_row_resident_truncated_vs_oracle(orc, lg, p):
    """The row-resident kernels (itft at every n, tft with n <= L/2; L <=
    2^14), batched, against the oracle at the truncation boundaries, with an
    all-(p-1) row."""
    L = 1 << lg
    B = 3
    sh = _tensors.stream_handle()
    for n in sorted({1, 2, L // 2 - 1, L // 2, L // 2 + 1, L - L // 5, L - 1, L}):
        x = orc.gen_u32(64, 0, lg * 100000 + n, B, n, p)
        x[1, :] = p - 1
        xt = torch.from_numpy(x.view(np.int32)).cuda()
        y = torch.empty((B, n), dtype=torch.int32, device="cuda")
        _native.check(_native.lib().mc_itft(xt.data_ptr(), y.data_ptr(), n, lg, B, p, sh))
        got = y.cpu().numpy().view(np.uint32)
        for r in range(B):
            assert np.array_equal(got[r], orc.itft(x[r], L, p)[0]), ("itft", L, n, r)
        for z in sorted({1, n // 3 + 1, n}):
            xz = torch.from_numpy(np.ascontiguousarray(x[:, :z]).view(np.int32)).cuda()
            t = torch.empty((B, n), dtype=torch.int32, device="cuda")
            _native.check(_native.lib().mc_tft(xz.data_ptr(), z, t.data_ptr(), n, lg, B, p, sh))
            got = t.cpu().numpy().view(np.uint32)
            for r in range(B):
                assert np.array_equal(got[r], orc.tft(x[r, :z], n, L, p)[0]), ("tft", L, n, z, r)
