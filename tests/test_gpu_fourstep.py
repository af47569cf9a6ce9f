"""GPU parity of the four-step large-transform path (configs 4 and 5) and the
three-primes CRT product, against the C oracle, the reference's golden pins
and size-independent evaluation identities."""

import hashlib

import numpy as np
import pytest
import torch

from conftest import P1, P2, P3

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc
    from gpu_helpers import eval_vec, gen_device, to_u32_np


@pytest.mark.parametrize("K", [14, 15, 16, 17, 18])
@pytest.mark.parametrize("p", [P1, P2, P3])
def test_fourstep_sizes_vs_oracle(orc, K, p):
    L = 1 << K
    for n in sorted({L, L - 1, L // 2 + 1, (3 * L) // 4 + 5}):
        for z1 in sorted({1, (n + 1) // 2, n - 7}):
            z2 = n + 1 - z1
            if z1 < 1 or z2 < 1:
                continue
            a = orc.gen_u32(40 + K, 0, n + z1, 2, z1, p)
            b = orc.gen_u32(40 + K, 1, n + z1, 2, z2, p)
            a[1, :] = p - 1
            b[1, :] = p - 1
            want, _, _ = orc.conv_batch(a, b, p, threads=8)
            at = torch.from_numpy(a.view(np.int32)).cuda()
            bt = torch.from_numpy(b.view(np.int32)).cuda()
            for eng in ("fft_pad", "tft"):
                got = to_u32_np(mc.conv_batch(at, bt, p, engine=eng))
                assert np.array_equal(got, want), (K, n, z1, eng)


@pytest.mark.parametrize("K", [14, 16, 19])
def test_fourstep_circular(orc, K):
    p = P3
    L = 1 << K
    u = orc.gen_u32(50, 0, K, 1, L, p)[0]
    v = orc.gen_u32(50, 1, K, 1, L, p)[0]
    fp = mc.FourierPrime.from_modulus(p)
    got = mc.circ_conv_fft(u.tolist(), v.tolist(), mc.ConvRequest(fp, engine="fft_pad"))
    # circular = linear folded mod x^L - 1
    lin, _, _ = orc.conv_batch(u[None], v[None], p, threads=8)
    lin = lin[0].astype(np.uint64)
    fold = lin[:L].copy()
    fold[: L - 1] = (fold[: L - 1] + lin[L:]) % p
    assert got == fold.tolist()


def test_cfg4_large_products(orc, golden_configs):
    """Config 4: 8 products of 2^22 x 2^22 mod 2013265921 (L = 2^23).
    Products 0 and 7 equal the reference's own poly_mul (sha256 pins made by
    tests/golden/make_golden.py --cfg4) and the oracle; all 8 pass the
    evaluation identity at two points."""
    p, z, B = P3, 1 << 22, 8
    a = gen_device(4, 0, 0, B, z, p)
    b = gen_device(4, 1, 0, B, z, p)
    c = mc.conv_batch(a, b, p, engine="fft_pad")
    torch.cuda.synchronize()
    pin = golden_configs["cfg4"]
    assert (pin["p"], pin["z1"], pin["z2"], pin["seed"]) == (p, z, z, 4)
    for rec in pin["rows"]:
        row = to_u32_np(c[rec["row"]])
        assert hashlib.sha256(row.tobytes()).hexdigest() == rec["sha256"], rec["row"]
        assert row[:8].tolist() == rec["head"] and row[-8:].tolist() == rec["tail"]
    for r in (0, B - 1):
        want, _, _ = orc.conv_batch(to_u32_np(a[r:r + 1]), to_u32_np(b[r:r + 1]), p)
        assert np.array_equal(to_u32_np(c[r:r + 1]), want), r
    for r in range(B):
        for x in (3, 1234567891 % p):
            assert eval_vec(c[r], x, p) == eval_vec(a[r], x, p) * eval_vec(b[r], x, p) % p, r


def test_cfg5_three_primes_pinned(golden_configs, orc):
    pin = golden_configs["cfg5"]
    z = pin["z"]
    a = gen_device(pin["seed"], 0, 0, 1, z, pin["hi"])[0]
    b = gen_device(pin["seed"], 1, 0, 1, z, pin["hi"])[0]
    limbs = mc.mul_three_primes_tensor(a, b)
    ln = to_u32_np(limbs)
    assert hashlib.sha256(ln.tobytes()).hexdigest() == pin["limbs_sha256"]
    assert [str(x) for x in orc.limbs_to_ints(ln[:, :4])] == pin["head"]
    assert [str(x) for x in orc.limbs_to_ints(ln[:, -4:])] == pin["tail"]
    # per-prime channels match the reference's per-prime products
    from paper_1609_01010_b200 import _native, _tensors

    for k, p in enumerate((P1, P2, P3)):
        r = torch.empty(2 * z - 1, dtype=torch.int32, device="cuda")
        _native.check(_native.lib().mc_mul_mod_prime_k(a.data_ptr(), z, b.data_ptr(), z,
                                                        r.data_ptr(), k,
                                                        _tensors.stream_handle()))
        assert hashlib.sha256(to_u32_np(r).tobytes()).hexdigest() == \
            pin["per_prime"][str(p)]["sha256"], p


@pytest.mark.parametrize("z1,z2", [(1 << 17, 1 << 17), (150001, 70001), (1 << 19, 1 << 18),
                                   (262139, 262147), (1 << 22, 1 << 22)])
def test_three_primes_fused_crt_path(orc, z1, z2):
    """Four-step sizes K = 18..23 run the fused path (inverse column passes of
    the three primes + Garner in one kernel): exact limbs vs the oracle,
    including unaligned operand lengths (no tensor-map loads) and the
    largest size p2's 2-adicity allows."""
    rng = np.random.default_rng(z1 ^ (z2 << 1))
    a = rng.integers(0, 1 << 30, z1, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 1 << 30, z2, dtype=np.uint64).astype(np.uint32)
    a[:5] = (1 << 30) - 1
    b[-5:] = (1 << 30) - 1
    at = torch.from_numpy(a.view(np.int32)).cuda()
    bt = torch.from_numpy(b.view(np.int32)).cuda()
    got = to_u32_np(mc.mul_three_primes_tensor(at, bt))
    want = orc.mul_three_primes(a, b, threads=8)
    assert np.array_equal(got, want), (z1, z2)


@pytest.mark.parametrize("z1,z2,off", [(1 << 20, 1 << 20, 0), (300007, 200003, 1),
                                        (1 << 21, 5, 0), (77, 1 << 21, 3)])
def test_three_primes_words_and_alignment(orc, z1, z2, off):
    """Four-step sizes with full 32-bit input words (reduced mod each prime
    on load), lopsided operands, and operands that are not 16-byte aligned
    (off words into a buffer: no tensor-map loads) -- exact limbs vs the
    oracle."""
    rng = np.random.default_rng(z1 + 3 * z2 + off)
    a = rng.integers(0, 1 << 32, z1, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 1 << 32, z2, dtype=np.uint64).astype(np.uint32)
    a[:3] = 0xFFFFFFFF
    b[-3:] = 0xFFFFFFFF
    abuf = torch.zeros(z1 + off, dtype=torch.int32, device="cuda")
    bbuf = torch.zeros(z2 + off, dtype=torch.int32, device="cuda")
    abuf[off:] = torch.from_numpy(a.view(np.int32)).cuda()
    bbuf[off:] = torch.from_numpy(b.view(np.int32)).cuda()
    got = to_u32_np(mc.mul_three_primes_tensor(abuf[off:], bbuf[off:]))
    want = orc.mul_three_primes(a, b, threads=8)
    assert np.array_equal(got, want), (z1, z2, off)


@pytest.mark.parametrize("z1,z2", [(1, 1), (1, 9), (5, 3), (300, 200), (4096, 4096),
                                    (5000, 3), (20000, 17000)])
def test_three_primes_small_exact(orc, z1, z2):
    rng = np.random.default_rng(z1 * 7 + z2)
    a = rng.integers(0, 1 << 30, z1, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 1 << 30, z2, dtype=np.uint64).astype(np.uint32)
    a[0] = (1 << 30) - 1
    b[-1] = (1 << 30) - 1
    got = mc.mul_three_primes(a.tolist(), b.tolist())
    want = orc.limbs_to_ints(orc.mul_three_primes(a, b))
    assert got == want
    if z1 * z2 <= 100000:
        exact = [0] * (z1 + z2 - 1)
        for i, x in enumerate(a.tolist()):
            for j, y in enumerate(b.tolist()):
                exact[i + j] += x * y
        assert got == exact


def test_crt3_kernel_edges(orc):
    n = 1000
    rng = np.random.default_rng(5)
    rs = [rng.integers(0, p, n, dtype=np.uint64).astype(np.uint32) for p in (P1, P2, P3)]
    for r, p in zip(rs, (P1, P2, P3)):
        r[:3] = [0, p - 1, 1]
    t = [torch.from_numpy(r.view(np.int32)).cuda() for r in rs]
    got = to_u32_np(mc.crt3(*t))
    assert np.array_equal(got, orc.crt3(*rs))


@pytest.mark.parametrize("z1,z2", [((1 << 19) + 1, 1 << 19), ((1 << 21) + 3, (1 << 20) + 5),
                                    (3_000_001, 1_194_304)])
def test_fourstep_truncated_large(orc, z1, z2):
    """Truncated (tft) engine past a power of two at L = 2^20..2^23: rows
    beyond NT*R/16 are never formed; bit-exact vs the oracle, and identical
    to the padded engine."""
    p = P3
    a = gen_device(70, 0, z1, 1, z1, p)
    b = gen_device(70, 1, z2, 1, z2, p)
    c = mc.conv_batch(a, b, p, engine="tft")
    want, _, _ = orc.conv_batch(to_u32_np(a), to_u32_np(b), p, orc.ENGINE_FFT_PAD)
    assert np.array_equal(to_u32_np(c), want)
    assert torch.equal(c, mc.conv_batch(a, b, p, engine="fft_pad"))


def test_beyond_2_24_vs_oracle(orc):
    """L = 2^25 (four-step with 2^13-point rows and 2^12-point columns), p1
    (2-adicity 26): bit-exact against the oracle, both engines."""
    p = P1
    z1, z2 = (1 << 24) + 1, 1 << 23
    a = orc.gen_u32(61, 0, 0, 1, z1, p)
    b = orc.gen_u32(61, 1, 0, 1, z2, p)
    a[0, :5] = p - 1
    b[0, -5:] = p - 1
    want, _, _ = orc.conv_batch(a, b, p)
    at = torch.from_numpy(a.view(np.int32)).cuda()
    bt = torch.from_numpy(b.view(np.int32)).cuda()
    for eng in ("fft_pad", "tft"):
        got = to_u32_np(mc.conv_batch(at, bt, p, engine=eng))
        assert np.array_equal(got, want), eng


@pytest.mark.parametrize("K,p", [(26, P1), (26, P3), (27, P3)])
def test_up_to_the_two_adicity(K, p):
    """L = 2^26 (four-step, 2^13 x 2^13) and 2^27 (level-scheduled fallback,
    p3 only) up to each prime's 2-adicity: evaluation identity at two points
    (the reference raises UnsupportedSizeError only beyond the 2-adicity)."""
    z1 = (1 << (K - 1)) + 3
    z2 = (1 << (K - 1)) - 7
    a = gen_device(62 + K, 0, 0, 1, z1, p)
    b = gen_device(62 + K, 1, 0, 1, z2, p)
    c = mc.conv_batch(a, b, p, engine="fft_pad")
    assert c.shape == (1, z1 + z2 - 1)
    for x in (3, 123456789):
        assert eval_vec(c, x, p) == eval_vec(a, x, p) * eval_vec(b, x, p) % p
    del c
    torch.cuda.empty_cache()


def test_beyond_the_two_adicity_raises():
    p = P2  # 2-adicity 23
    a = gen_device(70, 0, 0, 1, (1 << 22) + 1, p)
    with pytest.raises(mc.UnsupportedSizeError) as ei:
        mc.conv_batch(a, a, p)
    assert ei.value.required_two_adicity == 24


@pytest.mark.parametrize("K", [14, 16])
def test_row_prefetch_every_group(orc, K, monkeypatch):
    """The row pass's L2 prefetch (forced on: MC_ROW_PREFETCH=1) with two row
    groups per CTA at K = 14 (2^10-point rows) and one at K = 16: results
    unchanged, bit-exact vs the oracle."""
    monkeypatch.setenv("MC_ROW_PREFETCH", "1")
    p = P2
    n = (1 << K) - 3
    z1 = (n + 1) // 2
    a = orc.gen_u32(70 + K, 0, 0, 5, z1, p)
    b = orc.gen_u32(70 + K, 1, 0, 5, n + 1 - z1, p)
    want, _, _ = orc.conv_batch(a, b, p, threads=8)
    at = torch.from_numpy(a.view(np.int32)).cuda()
    bt = torch.from_numpy(b.view(np.int32)).cuda()
    got = to_u32_np(mc.conv_batch(at, bt, p, engine="fft_pad"))
    assert np.array_equal(got, want)
