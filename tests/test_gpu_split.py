"""GPU parity of the Eq. 13 split engine (nega_conv, circ_conv_split,
split_residues, recombine_residues; reference convolve.py:172-227) against
fixtures produced by the reference, plus the reference's own properties
(tests/test_convolve.py TestNegacyclic / TestSplitEngine, acceptance
criterion 8)."""

import numpy as np
import pytest
import torch

from conftest import P2, P3

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc


def test_golden_split_cases(golden_small):
    for c in golden_small["split"]:
        fp = mc.FourierPrime.from_modulus(c["p"])
        if c.get("poly"):
            cnt = mc.OpCounters()
            r = mc.poly_mul(mc.DensePoly(fp, tuple(c["u"])), mc.DensePoly(fp, tuple(c["v"])),
                            mc.ConvRequest(fp, engine="split", counters=cnt))
            assert list(r.coeffs) == c["out"], (c["p"], len(c["u"]), len(c["v"]))
            assert [cnt.butterflies, cnt.pointwise_muls] == c["counters"]
            continue
        cnt = mc.OpCounters()
        got = mc.circ_conv_split(c["u"], c["v"], mc.ConvRequest(fp, engine="split", counters=cnt))
        assert got == c["split"], (c["p"], c["size"])
        assert [cnt.butterflies, cnt.pointwise_muls] == c["split_counters"]
        a, b = mc.split_residues(c["u"], c["p"])
        assert (a, b) == (c["res_a"], c["res_b"])
        assert mc.recombine_residues(a, b, c["p"]) == c["recombined"] == c["u"]
        if "nega" in c:
            cn = mc.OpCounters()
            assert mc.nega_conv(c["u"], c["v"], mc.ConvRequest(fp, counters=cn)) == c["nega"]
            assert [cn.butterflies, cn.pointwise_muls] == c["nega_counters"]


def test_reference_properties(orc):
    fp17 = mc.FourierPrime.from_modulus(17)
    assert mc.nega_conv([0, 1], [0, 1], mc.ConvRequest(fp17)) == [16, 0]  # x^2 = -1
    assert mc.split_residues([1, 2, 3, 4], 17) == ([4, 6], [15, 15])
    fp = mc.FourierPrime.from_modulus(P2)
    rng = np.random.default_rng(8)
    for lg in range(1, 14):
        size = 1 << lg
        u = rng.integers(0, P2, size).tolist()
        v = rng.integers(0, P2, size).tolist()
        got = mc.circ_conv_split(u, v, mc.ConvRequest(fp))
        lin, _, _ = orc.conv_batch(np.array([u]), np.array([v]), P2)
        lin = lin[0].astype(np.uint64)
        circ = lin[:size].copy()
        circ[: size - 1] = (circ[: size - 1] + lin[size:]) % P2
        assert got == circ.tolist(), size
        delta = [1] + [0] * (size - 1)
        assert mc.circ_conv_split(delta, v, mc.ConvRequest(fp)) == v
        if lg <= 12:
            nega = mc.nega_conv(u, v, mc.ConvRequest(fp))
            full = lin.tolist() + [0]
            assert nega == [(full[i] - full[i + size]) % P2 for i in range(size)], size


def test_split_engine_poly_mul_agrees(orc):
    fp = mc.FourierPrime.from_modulus(P3)
    rng = np.random.default_rng(9)
    for z1, z2 in ((1, 1), (5, 3), (300, 200), (2049, 2048), (9000, 7000)):
        a = rng.integers(1, P3, z1).tolist()
        b = rng.integers(1, P3, z2).tolist()
        want, _, _ = orc.conv_batch(np.array([a]), np.array([b]), P3)
        r = mc.poly_mul(mc.DensePoly(fp, tuple(a)), mc.DensePoly(fp, tuple(b)),
                        mc.ConvRequest(fp, engine="split"))
        assert list(r.coeffs) == want[0].tolist()


def test_split_errors():
    fp17 = mc.FourierPrime.from_modulus(17)
    with pytest.raises(mc.UnsupportedSizeError):  # nega_conv at n = 16 needs 2^5
        mc.nega_conv([1] * 16, [1] * 16, mc.ConvRequest(fp17))
    with pytest.raises(ValueError):
        mc.circ_conv_split([1], [1], mc.ConvRequest(fp17))
    with pytest.raises(ValueError):
        mc.circ_conv_split([1, 2, 3], [4, 5, 6], mc.ConvRequest(fp17))
