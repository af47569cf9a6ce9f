"""Pin the C oracle (oracle/modconv_oracle.c) against fixtures produced by the
reference implementation itself (tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import P1, P2, P3


def _sha(a):
    return hashlib.sha256(np.asarray(a, dtype=np.uint32).tobytes()).hexdigest()


def _splitmix_np(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15))
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def test_generator_matches_numpy_restatement(orc):
    with np.errstate(over="ignore"):
        for seed, stream, row, hi in ((1, 0, 0, P1), (3, 1, 65535, P2), (5, 0, 7, 1 << 30)):
            key = _splitmix_np(_splitmix_np(_splitmix_np(np.uint64(seed)) ^ np.uint64(stream))
                               ^ np.uint64(row))
            v = _splitmix_np(key + np.arange(1000, dtype=np.uint64))
            want = (((v >> np.uint64(32)) * np.uint64(hi)) >> np.uint64(32)).astype(np.uint32)
            got = orc.gen_u32(seed, stream, row, 1, 1000, hi)[0]
            assert np.array_equal(got, want)
            assert got.max() < hi


def test_field_descriptors(orc, golden_small):
    for f in golden_small["fields"]:
        assert orc.two_adicity(f["p"]) == f["two_adicity"]
        assert orc.primitive_root(f["p"]) == f["generator"]
        for lg, w in f["roots"].items():
            assert orc.root_of_unity(f["p"], int(lg)) == w, (f["p"], lg)


def test_kats(orc, golden_small):
    k = golden_small["kats"]
    for case in k["dft_p5"]:
        y, _ = orc.moddft(case["x"], 5)
        assert y.tolist() == case["y"]
    assert [[1, 1, 1, 1], [4, 0, 0, 0], [1, 2, 4, 3]] == [c["y"] for c in k["dft_p5"]]
    t = k["tft_dc"]
    y, _ = orc.tft(t["x"], t["n"], t["L"], t["p"])
    assert y.tolist() == t["y"] == [9]
    for c in k["conv17"]:
        for eng, code in (("fft_pad", orc.ENGINE_FFT_PAD), ("tft", orc.ENGINE_TFT)):
            got, _, _ = orc.conv_batch(np.array([c["u"]]), np.array([c["v"]]), 17, code)
            assert got[0].tolist() == c[eng]
    assert k["conv17"][0]["tft"] == [3, 10, 8]
    assert k["modmul_2_60"]["value"] == 682155965


def test_transforms(orc, golden_small):
    for c in golden_small["transforms"]:
        p, L = c["p"], c["L"]
        if c["kind"] == "moddft":
            y, bf = orc.moddft(c["x"], p)
            assert y.tolist() == c["fwd"], (p, L)
            assert bf == c["butterflies"]
            y, _ = orc.moddft(c["x"], p, inverse=True)
            assert y.tolist() == c["inv"], (p, L)
        else:
            y, bf = orc.tft(c["x"], c["n"], L, p)
            assert y.tolist() == c["y"], (p, L, c["n"], len(c["x"]))
            assert bf == c["butterflies"]
            assert orc.tft_count(L, len(c["x"]), c["n"]) == bf
            y, bf = orc.itft(c["itft_in"], L, p)
            assert y.tolist() == c["itft_out"], (p, L, c["n"])
            assert bf == c["itft_butterflies"]
            assert orc.itft_count(L, c["n"]) == bf


def test_convolutions(orc, golden_small):
    for c in golden_small["convs"]:
        p = c["p"]
        if c.get("tag") == "all_p_minus_1":
            u = np.full(c["z1"], p - 1)
            v = np.full(c["z2"], p - 1)
        else:
            u, v = np.array(c["u"]), np.array(c["v"])
        for eng, code in (("fft_pad", orc.ENGINE_FFT_PAD), ("tft", orc.ENGINE_TFT)):
            got, bf, pw = orc.conv_batch(u[None], v[None], p, code)
            assert got[0].tolist() == c[eng], (p, len(u), len(v), eng)
            assert [bf, pw] == c[eng + "_counters"]


def test_config_rows(orc, golden_configs):
    for cfg in golden_configs["configs"]:
        p, z1, z2, seed = cfg["p"], cfg["z1"], cfg["z2"], cfg["seed"]
        code = orc.ENGINE_TFT if cfg["engine"] == "tft" else orc.ENGINE_FFT_PAD
        for rec in cfg["rows"]:
            a = orc.gen_u32(seed, 0, rec["row"], 1, z1, p)
            b = orc.gen_u32(seed, 1, rec["row"], 1, z2, p)
            c, bf, pw = orc.conv_batch(a, b, p, code)
            assert _sha(c[0]) == rec["sha256"], (cfg["cfg"], rec["row"])
            assert [bf, pw] == rec["counters"]


def test_cfg5_three_primes(orc, golden_configs):
    pin = golden_configs.get("cfg5")
    if pin is None:
        pytest.skip("cfg5 pin not generated (make_golden.py --cfg5)")
    z = pin["z"]
    a = orc.gen_u32(pin["seed"], 0, 0, 1, z, pin["hi"])[0]
    b = orc.gen_u32(pin["seed"], 1, 0, 1, z, pin["hi"])[0]
    limbs = orc.mul_three_primes(a, b)
    assert hashlib.sha256(limbs.tobytes()).hexdigest() == pin["limbs_sha256"]
    ints = orc.limbs_to_ints(limbs[:, :4])
    assert [str(x) for x in ints] == pin["head"]


def test_crt_small_exact(orc):
    rng = np.random.default_rng(7)
    a = rng.integers(0, 1 << 30, 300, dtype=np.uint64)
    b = rng.integers(0, 1 << 30, 200, dtype=np.uint64)
    limbs = orc.mul_three_primes(a, b)
    want = [0] * 499
    for i, x in enumerate(a.tolist()):
        for j, y in enumerate(b.tolist()):
            want[i + j] += x * y
    assert orc.limbs_to_ints(limbs) == want


def test_eval_homomorphism_helper(orc):
    a = orc.gen_u32(9, 0, 0, 3, 50, P2)
    b = orc.gen_u32(9, 1, 0, 3, 40, P2)
    c, _, _ = orc.conv_batch(a, b, P2)
    x = np.array([3, 12345, P2 - 1])
    lhs = orc.eval_mod(c, x, P2)
    rhs = orc.eval_mod(a, x, P2) * orc.eval_mod(b, x, P2) % np.uint64(P2)
    assert np.array_equal(lhs, rhs)
