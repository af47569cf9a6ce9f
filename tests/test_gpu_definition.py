"""GPU parity of the definition engine (mc_conv_direct: the defining sum,
any field, any length) and of the reference API entries built on it:
lin_conv_def / circ_conv_def (convolve.py:54-87), mul_schoolbook /
mul_karatsuba / eval_poly (poly.py:90-181), poly_mul(engine="definition")
beyond the field's 2-adicity, conv_batch(engine="definition"), and the
transform variants moddft_naive / dft_basecase / moddft_plan
(transform.py:199-376).  Known answers re-derived from the reference's
tests (tests/test_convolve.py:33-75, tests/test_poly.py, tests/test_cli.py:
171-178); random cases against exact integer convolution."""

import numpy as np
import pytest
import torch

from conftest import P2, P3

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc


def _exact_lin(u, v, p):
    out = [0] * (len(u) + len(v) - 1)
    for i, x in enumerate(u):
        if x:
            for j, y in enumerate(v):
                out[i + j] += x * y
    return [c % p for c in out]


def _exact_circ(u, v, p):
    n = len(u)
    out = [0] * n
    for i in range(n):
        for j in range(n):
            out[(i + j) % n] += u[i] * v[j]
    return [c % p for c in out]


def test_definition_kats():
    fp5, fp7, fp17, fp257 = (mc.FourierPrime.from_modulus(q) for q in (5, 7, 17, 257))
    v = [1, 2, 3, 4]
    assert mc.circ_conv_def([1, 0, 0, 0], v, fp17) == v
    assert mc.circ_conv_def([0, 1, 0, 0], [1, 2, 3, 4], fp17) == [4, 1, 2, 3]
    assert mc.circ_conv_def([1, 1, 1, 1], [1, 2, 3, 4], fp5) == [0, 0, 0, 0]
    assert mc.lin_conv_def([1], v, fp17) == v
    assert mc.lin_conv_def([1, 2], [3, 4], fp7) == [3, 3, 1]  # p = 7: no 4th root of unity
    rng = np.random.default_rng(5)
    u = rng.integers(0, 257, 9).tolist()
    w = rng.integers(0, 257, 9).tolist()
    assert mc.circ_conv_def(u, w, fp257) == _exact_circ(u, w, 257)
    with pytest.raises(ValueError):
        mc.circ_conv_def([1, 2], [1], fp17)
    with pytest.raises(ValueError):
        mc.lin_conv_def([], [1], fp17)


@pytest.mark.parametrize("p", [7, 17, 257, 65537, P2, P3])
def test_definition_random_vs_exact(p):
    """Lengths across tile boundaries (256 outputs per CTA), all-(p-1) rows
    (largest partial sums), circular and linear."""
    fp = mc.FourierPrime.from_modulus(p)
    rng = np.random.default_rng(p % 1000)
    for z1, z2 in ((1, 1), (1, 300), (255, 2), (256, 257), (513, 700), (1000, 31)):
        u = rng.integers(0, p, z1).tolist()
        v = rng.integers(0, p, z2).tolist()
        assert mc.lin_conv_def(u, v, fp) == _exact_lin(u, v, p), (p, z1, z2)
    top = [p - 1] * 600
    assert mc.lin_conv_def(top, top, fp) == _exact_lin(top, top, p)
    for n in (1, 3, 256, 300):
        u = rng.integers(0, p, n).tolist()
        v = rng.integers(0, p, n).tolist()
        assert mc.circ_conv_def(u, v, fp) == _exact_circ(u, v, p), (p, n)


def test_poly_mul_definition_beyond_two_adicity():
    """The reference's definition engine keeps working where no transform
    exists (p = 17 has 2-adicity 4: products longer than 16)."""
    fp = mc.FourierPrime.from_modulus(17)
    rng = np.random.default_rng(17)
    a = mc.DensePoly(fp, tuple(rng.integers(1, 17, 40).tolist()))
    b = mc.DensePoly(fp, tuple(rng.integers(1, 17, 25).tolist()))
    cnt = mc.OpCounters()
    got = mc.poly_mul(a, b, mc.ConvRequest(fp, engine="definition", counters=cnt))
    assert list(got.coeffs) == _exact_lin(list(a.coeffs), list(b.coeffs), 17)
    assert (cnt.butterflies, cnt.pointwise_muls) == (0, 0)
    with pytest.raises(mc.UnsupportedSizeError):
        mc.poly_mul(a, b, mc.ConvRequest(fp, engine="tft"))
    # inside the 2-adicity both routes agree
    fp2 = mc.FourierPrime.from_modulus(P2)
    a2 = mc.DensePoly(fp2, tuple(rng.integers(0, P2, 100).tolist()))
    b2 = mc.DensePoly(fp2, tuple(rng.integers(0, P2, 77).tolist()))
    assert (mc.poly_mul(a2, b2, mc.ConvRequest(fp2, engine="definition"))
            == mc.poly_mul(a2, b2, mc.ConvRequest(fp2, engine="tft")))


def test_schoolbook_karatsuba_eval():
    fp = mc.FourierPrime.from_modulus(P2)
    rng = np.random.default_rng(3)
    a = mc.DensePoly(fp, tuple(rng.integers(0, P2, 50).tolist()) + (0, 0))  # trailing zeros kept
    b = mc.DensePoly(fp, tuple(rng.integers(0, P2, 33).tolist()))
    want = _exact_lin(list(a.coeffs), list(b.coeffs), P2)
    s = mc.mul_schoolbook(a, b)
    assert list(s.coeffs) == want and len(s.coeffs) == 52 + 33 - 1  # not normalized
    assert mc.mul_karatsuba(a, b) == s
    assert mc.mul_karatsuba(a, b, threshold=1) == s
    with pytest.raises(ValueError):
        mc.mul_karatsuba(a, b, threshold=0)
    assert mc.mul_schoolbook(a, mc.DensePoly.zero(fp)).coeffs == ()
    other = mc.DensePoly(mc.FourierPrime.from_modulus(17), (1,))
    with pytest.raises(mc.FieldMismatchError):
        mc.mul_schoolbook(a, other)
    x = mc.Felt(12345, fp)
    ev = lambda poly: sum(c * pow(12345, i, P2) for i, c in enumerate(poly.coeffs)) % P2
    assert mc.eval_poly(s, x).value == ev(s) == ev(a) * ev(b) % P2
    with pytest.raises(mc.FieldMismatchError):
        mc.eval_poly(a, mc.Felt(1, mc.FourierPrime.from_modulus(17)))
    with pytest.raises(ValueError):
        mc.Felt(P2, fp)
    assert (mc.Felt(3, fp) * mc.Felt(3, fp).inv()).value == 1


def test_conv_batch_definition(orc):
    p = P3
    B, z1, z2 = 70, 300, 211
    a = orc.gen_u32(71, 0, 0, B, z1, p)
    b = orc.gen_u32(71, 1, 0, B, z2, p)
    want = orc.conv_batch(a, b, p, orc.ENGINE_FFT_PAD, threads=8)[0]
    at = torch.from_numpy(a.view(np.int32))
    bt = torch.from_numpy(b.view(np.int32))
    got = mc.conv_batch(at.cuda(), bt.cuda(), p, engine="definition")
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want)
    got_h = mc.conv_batch(at, bt, p, engine="definition")  # host tensors
    assert np.array_equal(got_h.numpy().view(np.uint32), want)


def test_transform_variants():
    fp = mc.FourierPrime.from_modulus(P2)
    rng = np.random.default_rng(8)
    for L in (2, 4, 8):
        t = mc.get_table(fp, L)
        x = rng.integers(0, P2, L).tolist()
        want = mc.moddft(x, t)
        cnt = mc.OpCounters()
        assert mc.dft_basecase(x, t, "fwd", cnt) == want
        assert cnt.butterflies == {2: 1, 4: 4, 8: 12}[L]
        assert mc.dft_basecase(want, t, "inv") == x
        assert mc.moddft_naive(x, t) == want
    t = mc.get_table(fp, 64)
    x = rng.integers(0, P2, 64).tolist()
    want = mc.moddft(x, t)
    for splits, base in (((2, 4), 8), ((8,), 8), ((2, 2, 2, 2, 2), 2), ((4, 4), 4)):
        cnt = mc.OpCounters()
        assert mc.moddft_plan(x, t, splits, base, "fwd", cnt) == want
        assert cnt.butterflies == 32 * 6
    assert mc.moddft_plan(want, t, (8,), 8, "inv") == x
    for bad in (((3,), 8), ((8,), 16), ((8,), 4)):
        with pytest.raises(ValueError):
            mc.moddft_plan(x, t, *bad)
    with pytest.raises(ValueError):
        mc.dft_basecase(x[:16], mc.get_table(fp, 16))
    with pytest.raises(ValueError):
        mc.dft_basecase(x[:4], mc.get_table(fp, 8))
