"""CPU-only tests: host-side mirror of the reference API, analytic
OpCounters, error mapping, and that the C-ABI library loads and exports
every symbol include/modconv_b200.h declares (no compute without a GPU)."""

import ctypes
import os
import re

import pytest

from conftest import P1, P2, P3, REPO

import paper_1609_01010_b200 as mc
from paper_1609_01010_b200 import _native
from paper_1609_01010_b200.transform import full_count, itft_count, tft_count


def _header_symbols():
    src = open(os.path.join(REPO, "include", "modconv_b200.h")).read()
    return sorted(set(re.findall(r"\b(mc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    lib = _native.lib()
    declared = _header_symbols()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
    # the Python binding covers every declared entry point
    assert set(declared) <= set(_native.EXPORTED)
    assert lib.mc_version().startswith(b"modconv_b200")


def test_field_info_and_roots_match_reference(golden_small):
    lib = _native.lib()
    for f in golden_small["fields"]:
        a, g = ctypes.c_int(), ctypes.c_uint32()
        assert lib.mc_field_info(f["p"], ctypes.byref(a), ctypes.byref(g)) == 0
        assert (a.value, g.value) == (f["two_adicity"], f["generator"])
        fp = mc.FourierPrime.from_modulus(f["p"])
        assert (fp.two_adicity, fp.generator) == (f["two_adicity"], f["generator"])
        for lg, w in f["roots"].items():
            r = ctypes.c_uint32()
            assert lib.mc_root_of_unity(f["p"], int(lg), ctypes.byref(r)) == 0
            assert r.value == w
            assert mc.root_of_unity(fp, 1 << int(lg)).value == w


def test_unsupported_size_error_carries_adicity():
    lib = _native.lib()
    r = ctypes.c_uint32()
    assert lib.mc_root_of_unity(17, 5, ctypes.byref(r)) == _native.MC_EUNSUPPORTED
    assert lib.mc_last_required_two_adicity() == 5
    with pytest.raises(mc.UnsupportedSizeError) as e:
        _native.check(_native.MC_EUNSUPPORTED)
    assert e.value.required_two_adicity == 5
    assert isinstance(e.value, ValueError)
    fp17 = mc.FourierPrime.from_modulus(17)
    with pytest.raises(mc.UnsupportedSizeError) as e:
        mc.root_of_unity(fp17, 32)
    assert e.value.required_two_adicity == 5
    with pytest.raises(mc.UnsupportedSizeError):
        mc.get_table(fp17, 32)
    with pytest.raises(ValueError):
        mc.get_table(fp17, 12)


def test_invalid_field():
    lib = _native.lib()
    assert lib.mc_field_info(15, None, None) == _native.MC_EINVAL
    with pytest.raises(ValueError):
        mc.FourierPrime.from_modulus(15)
    with pytest.raises(ValueError):
        mc.FourierPrime(17, 3, 3)
    with pytest.raises(ValueError):
        mc.FourierPrime(17, 4, 4)
    # moduli above 2^31 are valid fields but not GPU-hostable
    fp = mc.FourierPrime.from_modulus(4611686018427387847)
    with pytest.raises(mc.UnsupportedSizeError):
        from paper_1609_01010_b200.field import check_transform_size

        check_transform_size(fp, 1)
    assert mc.FourierPrime.from_modulus(2**31 - 1).two_adicity == 1


def test_conv_request_validation():
    fp = mc.FourierPrime.from_modulus(P2)
    with pytest.raises(ValueError):
        mc.ConvRequest(fp, engine="fancy")
    with pytest.raises(ValueError):
        mc.ConvRequest(fp, threads=0)
    assert mc.ENGINES == ("definition", "fft_pad", "tft", "split", "auto")


def test_poly_mul_host_paths_without_gpu():
    """Field checks and the zero short-circuit happen before any device work."""
    fp17 = mc.FourierPrime.from_modulus(17)
    fp257 = mc.FourierPrime.from_modulus(257)
    with pytest.raises(mc.FieldMismatchError):
        mc.poly_mul(mc.DensePoly.one(fp17), mc.DensePoly.one(fp257), mc.ConvRequest(fp17))
    with pytest.raises(mc.FieldMismatchError):
        mc.poly_mul(mc.DensePoly.one(fp17), mc.DensePoly.one(fp17), mc.ConvRequest(fp257))
    cnt = mc.OpCounters()
    z = mc.poly_mul(mc.DensePoly.zero(fp17), mc.DensePoly(fp17, (1, 2)),
                    mc.ConvRequest(fp17, engine="tft", counters=cnt))
    assert z.is_zero() and cnt == mc.OpCounters()
    with pytest.raises(ValueError):
        mc.poly_mul(mc.DensePoly.one(fp17), mc.DensePoly.one(fp17),
                    mc.ConvRequest(fp17, engine="auto"))


def test_dense_poly_semantics():
    fp = mc.FourierPrime.from_modulus(17)
    with pytest.raises(ValueError):
        mc.DensePoly(fp, (17,))
    assert mc.DensePoly.from_ints(fp, [20, -1]).coeffs == (3, 16)
    a = mc.DensePoly(fp, (1, 2, 0, 0))
    assert a.degree() == 1 and a.normalize().coeffs == (1, 2)
    assert mc.DensePoly(fp, (0, 0)).normalize() == mc.DensePoly.zero(fp)
    b = mc.DensePoly(fp, (1, 2))
    assert b.normalize() is b


def test_analytic_counters_match_reference(golden_small, golden_configs):
    for c in golden_small["convs"]:
        z1 = c.get("z1", len(c.get("u", [])))
        z2 = c.get("z2", len(c.get("v", [])))
        for eng in ("fft_pad", "tft"):
            cnt = mc.OpCounters()
            from paper_1609_01010_b200.convolve import count_engine

            count_engine(eng, z1, z2, cnt)
            assert [cnt.butterflies, cnt.pointwise_muls] == c[eng + "_counters"], (z1, z2, eng)
    for c in golden_small["transforms"]:
        if c["kind"] == "moddft":
            assert full_count(c["L"]) == c["butterflies"]
        else:
            assert tft_count(c["L"], len(c["x"]), c["n"]) == c["butterflies"]
            assert itft_count(c["L"], c["n"]) == c["itft_butterflies"]
    for cfg in golden_configs["configs"]:
        from paper_1609_01010_b200.convolve import count_engine

        cnt = mc.OpCounters()
        count_engine(cfg["engine"], cfg["z1"], cfg["z2"], cnt)
        assert [cnt.butterflies, cnt.pointwise_muls] == cfg["rows"][0]["counters"]


def test_truncated_bounds_hold_analytically():
    """n*log2(L)/2 + L bound (reference tests/test_acceptance.py:147-167)."""
    for lg in range(1, 11):
        L = 1 << lg
        for n in range(1, L + 1):
            bound = n * lg / 2 + L
            assert tft_count(L, n, n) <= bound
            assert itft_count(L, n) <= bound


def test_compute_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    fp = mc.FourierPrime.from_modulus(P3)
    with pytest.raises(RuntimeError, match="CUDA"):
        mc.conv_tft([1, 2], [3, 4], mc.ConvRequest(fp, engine="tft"))
    with pytest.raises(RuntimeError, match="CUDA"):
        mc.conv_batch(torch.zeros((2, 3), dtype=torch.int32), torch.zeros((2, 3),
                      dtype=torch.int32), fp)


def test_kernel_model_matches_oracle(orc):
    """The position-level model of the fused kernel's relaxed truncated
    schedule (tests/kernel_model.py) reproduces the oracle exactly."""
    import random

    import kernel_model as km

    for p in (257, P2, P3, P1):
        rng = random.Random(p)
        for z1, z2 in [(1, 1), (3, 5), (8, 9), (17, 17), (30, 50), (100, 28), (187, 262),
                       (129, 128)]:
            n = z1 + z2 - 1
            if (n - 1).bit_length() > orc.two_adicity(p):
                continue
            u = [rng.randrange(p) for _ in range(z1)]
            v = [rng.randrange(p) for _ in range(z2)]
            got, _ = km.conv_tft_model(u, v, p, lambda L: orc.root_of_unity(p, L.bit_length() - 1))
            assert got == orc.schoolbook(u, v, p), (p, z1, z2)


def test_factorization_large_safe_prime_is_fast():
    """Primitive roots come from a rho factorization (field.py:61-95): a
    62-bit safe prime's descriptor is built at once (trial division of p-1
    would take ~2^30 steps)."""
    import time

    from paper_1609_01010_b200.field import factorize

    t0 = time.perf_counter()
    fp = mc.FourierPrime.from_modulus(2305843009213699919)
    assert time.perf_counter() - t0 < 1.0
    assert (fp.two_adicity, fp.generator) == (1, 13)
    assert factorize(2305843009213699918) == (2, 1152921504606849959)
    assert factorize(1) == ()
    assert factorize(2**4 * 3**3 * 1000003 * 998244353) == (2, 3, 1000003, 998244353)
    assert factorize((2**31 - 1) * (2**31 - 19)) == (2**31 - 19, 2**31 - 1)


def test_large_field_rejected_before_any_work():
    """conv_batch on a field the 32-bit kernels cannot host raises
    UnsupportedSizeError at once (no hang, no device needed)."""
    import torch

    fp = mc.FourierPrime.from_modulus(2305843009213699919)
    one = torch.ones((1, 1), dtype=torch.int32)
    with pytest.raises(mc.UnsupportedSizeError):
        mc.conv_batch(one, one, fp, engine="fft_pad")
    with pytest.raises(mc.UnsupportedSizeError) as e:
        mc.conv_batch(torch.ones((1, 3), dtype=torch.int32), one.repeat(1, 2), fp)
    assert e.value.required_two_adicity == 2


def test_felt_constructors():
    """FourierPrime.felt / zero / one (field.py:140-150)."""
    fp = mc.FourierPrime.from_modulus(P3)
    assert fp.felt(-1).value == P3 - 1
    assert fp.felt(P3 + 5).value == 5
    assert fp.zero().value == 0 and fp.one().value == 1
    assert (fp.one() + fp.felt(-1)) == fp.zero()


def test_foreign_field_keeps_its_generator():
    """A duck-typed field (the reference's FourierPrime) keeps its generator:
    FourierPrime(17, 4, 5) has w_16 = 5, not the smallest root's 3."""

    class Foreign:
        p, two_adicity, generator = 17, 4, 5

    from paper_1609_01010_b200.field import as_field

    fp = as_field(Foreign())
    assert fp.generator == 5
    assert mc.root_of_unity(fp, 16).value == 5
    assert mc.root_of_unity(as_field(17), 16).value == 3
    with pytest.raises(ValueError):
        class Bad:
            p, two_adicity, generator = 17, 4, 4

        as_field(Bad())


def test_use_generator_validates():
    lib = _native.lib()
    assert lib.mc_use_generator(17, 4) == _native.MC_EINVAL  # order 4, not primitive
    assert lib.mc_use_generator(15, 2) == _native.MC_EINVAL
    assert lib.mc_use_generator(17, 5) == 0
    r = ctypes.c_uint32()
    assert lib.mc_root_of_unity(17, 4, ctypes.byref(r)) == 0 and r.value == 5
    assert lib.mc_use_generator(17, 0) == 0
    assert lib.mc_root_of_unity(17, 4, ctypes.byref(r)) == 0 and r.value == 3
