"""GPU tests of the boundary types: fields with a non-smallest generator
(reference-generated fixtures), poly_mul returning the caller's own
DensePoly class and field (convolve.py:277-278, 296), split_residues /
recombine_residues at any length (convolve.py:214-227), and the stream=
argument of the tensor APIs."""

import json
import os
from dataclasses import dataclass

import numpy as np
import pytest
import torch

from conftest import GOLDEN, P2, P3

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc


@pytest.fixture(scope="module")
def gen_cases():
    with open(os.path.join(GOLDEN, "reference_generators.json")) as f:
        return json.load(f)["cases"]


def test_transforms_with_caller_generator(gen_cases):
    """moddft / tft / itft use the field's own generator, as the reference's
    TwiddleTable does (transform.py:83): FourierPrime(17, 4, 5) and others."""
    for c in gen_cases:
        p, g, L = c["p"], c["g"], c["L"]
        fp = mc.FourierPrime(p, mc.FourierPrime.from_modulus(p).two_adicity, g)
        t = mc.TwiddleTable(fp, L)
        assert t.root == c["root"]
        assert mc.moddft(c["x"], t, "fwd") == c["fwd"], (p, g, L)
        assert mc.moddft(c["x"], t, "inv") == c["inv"], (p, g, L)
        c1, c2 = mc.OpCounters(), mc.OpCounters()
        assert mc.tft(t, c["tft_in"], c["n"], c1) == c["tft_out"], (p, g, L)
        assert mc.itft(t, c["tft_out"], c2) == c["itft_out"], (p, g, L)
        assert [c1.butterflies, c2.butterflies] == c["counters"]
        # the smallest-root table for the same (p, L) is still served alongside
        t0 = mc.get_table(mc.FourierPrime.from_modulus(p), L)
        y0 = mc.moddft(c["x"], t0, "fwd")
        if t0.root != t.root:
            assert y0 != c["fwd"]
        assert mc.moddft(y0, t0, "inv") == c["x"]


@dataclass(frozen=True)
class ForeignField:  # shaped like the reference's FourierPrime
    p: int
    two_adicity: int
    generator: int


@dataclass(frozen=True)
class ForeignPoly:  # shaped like the reference's DensePoly
    field: ForeignField
    coeffs: tuple

    @classmethod
    def zero(cls, field):
        return cls(field, ())

    def normalize(self):
        c = list(self.coeffs)
        while c and not c[-1]:
            c.pop()
        return ForeignPoly(self.field, tuple(c))


@pytest.mark.parametrize("engine", ["fft_pad", "tft", "definition", "split"])
def test_poly_mul_returns_callers_class(engine):
    ref = mc.FourierPrime.from_modulus(P2)
    ff = ForeignField(P2, ref.two_adicity, ref.generator)
    rng = np.random.default_rng(11)
    u = tuple(int(x) for x in rng.integers(0, P2, 37))
    v = tuple(int(x) for x in rng.integers(0, P2, 23)) + (0, 0)
    r = mc.poly_mul(ForeignPoly(ff, u), ForeignPoly(ff, v), mc.ConvRequest(ff, engine=engine))
    assert type(r) is ForeignPoly and r.field is ff
    want = mc.poly_mul(mc.DensePoly(ref, u), mc.DensePoly(ref, v),
                       mc.ConvRequest(ref, engine=engine))
    assert r.coeffs == want.coeffs
    assert r == ForeignPoly(ff, want.coeffs)
    z = mc.poly_mul(ForeignPoly(ff, (0, 0)), ForeignPoly(ff, v), mc.ConvRequest(ff, engine=engine))
    assert z == ForeignPoly(ff, ())
    # this package's own class keeps the operands' field object
    own = mc.poly_mul(mc.DensePoly(ref, u), mc.DensePoly(ref, v),
                      mc.ConvRequest(ref, engine=engine))
    assert own.field is ref


@pytest.mark.parametrize("size", [0, 1, 2, 3, 6, 7, 10, 12, 64, 100, 4097])
def test_split_residues_any_length(size):
    p = P3
    rng = np.random.default_rng(size)
    u = [int(x) for x in rng.integers(0, p, size)]
    n = size >> 1
    a, b = mc.split_residues(u, p)
    assert a == [(u[j] + u[j + n]) % p for j in range(n)]
    assert b == [(u[j] - u[j + n]) % p for j in range(n)]
    inv2 = (p + 1) >> 1
    w = mc.recombine_residues(a, b, p)
    assert w == [(x + y) * inv2 % p for x, y in zip(a, b)] + \
        [(x - y) * inv2 % p for x, y in zip(a, b)]
    assert w == u[:2 * n]
    # unequal halves pair up to the shorter one, like zip
    assert mc.recombine_residues(a + [5], b, p) == w


def test_stream_argument_is_stream_safe(orc):
    """conv_batch / mul_three_primes_tensor with stream=: temporaries and the
    output are allocated on that stream and the result is right after the
    stream is synchronized, while the current stream is busy elsewhere."""
    p = P3
    a = orc.gen_u32(91, 0, 0, 64, 1500, p)
    b = orc.gen_u32(91, 1, 0, 64, 2100, p)
    want, _, _ = orc.conv_batch(a, b, p, threads=8)
    at = torch.from_numpy(a.view(np.int32)).cuda()
    bt = torch.from_numpy(b.view(np.int32)).cuda()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    outs = []
    for k in range(8):
        # a strided view forces a contiguous temporary inside the call
        at_s = torch.cat([at, at], dim=1)[:, :1500] if k % 2 else at
        outs.append(mc.conv_batch(at_s, bt, p, engine="tft", stream=s))
    big = torch.empty(1 << 26, dtype=torch.int32, device="cuda")
    big.fill_(7)  # churn the current stream's allocator while s runs
    s.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy().view(np.uint32), want)
    x = torch.from_numpy(orc.gen_u32(92, 0, 0, 1, 3000, 1 << 30)[0].view(np.int32)).cuda()
    y = torch.from_numpy(orc.gen_u32(92, 1, 0, 1, 2000, 1 << 30)[0].view(np.int32)).cuda()
    s.wait_stream(torch.cuda.current_stream())
    limbs = mc.mul_three_primes_tensor(x, y, stream=s)
    s.synchronize()
    want3 = orc.mul_three_primes(x.cpu().numpy().view(np.uint32), y.cpu().numpy().view(np.uint32))
    assert np.array_equal(limbs.cpu().numpy().view(np.uint32), want3)
