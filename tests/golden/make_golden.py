"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --cfg5     # + config-5 pin (~2 min)
    python tests/golden/make_golden.py --cfg4     # + config-4 pin (rows 0 and 7, ~8 min)

It imports the unmodified reference package `modconv` from
/root/reference/pkg/src and records its outputs for seeded inputs built with
the shared generator (oracle.gen_u32 -- splitmix64, index addressable), so the
fixtures store seeds plus outputs (full vectors for small cases, sha256 of the
little-endian uint32 output plus a few coefficients for the BASELINE configs).
The committed JSON files are what the tests read; /root/reference is never
read at test time.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import modconv  # noqa: E402  (the reference)
from modconv import (  # noqa: E402
    ConvRequest,
    DensePoly,
    FourierPrime,
    OpCounters,
    get_table,
    itft,
    moddft,
    poly_mul,
    tft,
)
from modconv.convolve import (  # noqa: E402
    circ_conv_split,
    conv_tft,
    lin_conv_fft_pad,
    nega_conv,
    recombine_residues,
    split_residues,
)

from oracle import oracle  # noqa: E402  (only for the shared input generator)

P1, P2, P3 = 469762049, 998244353, 2013265921


def sha(vals) -> str:
    return hashlib.sha256(np.asarray(vals, dtype=np.uint32).tobytes()).hexdigest()


def fields():
    out = []
    for p in (5, 17, 257, 7681, 12289, 65537, 786433, P1, P2, P3):
        fp = FourierPrime.from_modulus(p)
        roots = {}
        for lg in range(0, min(fp.two_adicity, 24) + 1):
            roots[str(lg)] = modconv.root_of_unity(fp, 1 << lg).value
        out.append({"p": p, "two_adicity": fp.two_adicity, "generator": fp.generator,
                    "roots": roots})
    return out


def kats():
    fp5 = FourierPrime.from_modulus(5)
    fp17 = FourierPrime.from_modulus(17)
    t4 = get_table(fp5, 4)
    out = {
        "dft_p5": [
            {"x": x, "y": moddft(x, t4)} for x in ([1, 0, 0, 0], [1, 1, 1, 1], [0, 1, 0, 0])
        ],
        "tft_dc": {"p": 17, "L": 4, "x": [9], "n": 1, "y": tft(get_table(fp17, 4), [9], 1)},
        "conv17": [
            {"u": [1, 2], "v": [3, 4], "tft": conv_tft([1, 2], [3, 4], ConvRequest(fp17, "tft")),
             "fft_pad": lin_conv_fft_pad([1, 2], [3, 4], ConvRequest(fp17, "fft_pad"))},
            {"u": [5], "v": [7], "tft": conv_tft([5], [7], ConvRequest(fp17, "tft")),
             "fft_pad": lin_conv_fft_pad([5], [7], ConvRequest(fp17, "fft_pad"))},
        ],
        "modmul_2_60": {"p": P2, "value": (2**30 % P2) * (2**30 % P2) % P2},
    }
    return out


def transforms(rng):
    cases = []
    for p in (257, 7681, P2, P1, P3):
        fp = FourierPrime.from_modulus(p)
        for lg in range(0, min(fp.two_adicity, 10) + 1):
            L = 1 << lg
            t = get_table(fp, L)
            x = [rng.randrange(p) for _ in range(L)]
            c1, c2 = OpCounters(), OpCounters()
            cases.append({"kind": "moddft", "p": p, "L": L, "x": x,
                          "fwd": moddft(x, t, "fwd", c1), "inv": moddft(x, t, "inv", c2),
                          "butterflies": c1.butterflies})
    for p in (257, P2, P1, P3):
        fp = FourierPrime.from_modulus(p)
        for L in (1, 2, 4, 8, 16, 32, 64, 256):
            if L.bit_length() - 1 > fp.two_adicity:
                continue
            t = get_table(fp, L)
            ns = sorted({1, 2, L // 2, L // 2 + 1, L - 1, L, max(1, (3 * L) // 4 + 1)})
            for n in ns:
                if not 1 <= n <= L:
                    continue
                for z in sorted({1, n, max(1, n // 2), max(1, (n * 5) // 7)}):
                    x = [rng.randrange(p) for _ in range(z)]
                    fc = OpCounters()
                    spec = tft(t, x, n, fc)
                    xs = [rng.randrange(p) for _ in range(n)]
                    ic = OpCounters()
                    back = itft(t, xs, ic)
                    cases.append({"kind": "tft", "p": p, "L": L, "n": n, "x": x, "y": spec,
                                  "butterflies": fc.butterflies,
                                  "itft_in": xs, "itft_out": back,
                                  "itft_butterflies": ic.butterflies})
    return cases


def convs(rng):
    cases = []
    for p in (17, 257, P2, P1, P3):
        fp = FourierPrime.from_modulus(p)
        sizes = [(1, 1), (1, 5), (2, 2), (3, 7), (16, 16), (17, 17), (33, 31), (64, 3),
                 (100, 100), (128, 128), (129, 1), (200, 57)]
        if p == P3:
            sizes += [(513, 512), (1000, 700)]
        for z1, z2 in sizes:
            n = z1 + z2 - 1
            if (n - 1).bit_length() > fp.two_adicity:
                continue
            u = [rng.randrange(p) for _ in range(z1)]
            v = [rng.randrange(p) for _ in range(z2)]
            entry = {"p": p, "u": u, "v": v}
            for eng, fn in (("fft_pad", lin_conv_fft_pad), ("tft", conv_tft)):
                cnt = OpCounters()
                entry[eng] = fn(u, v, ConvRequest(fp, engine=eng, counters=cnt))
                entry[eng + "_counters"] = [cnt.butterflies, cnt.pointwise_muls]
            cases.append(entry)
    # edge vectors: all p-1 operands (maximal lazy ranges), zeros
    for p in (P1, P2, P3):
        fp = FourierPrime.from_modulus(p)
        for z1, z2 in ((1024, 1024), (1500, 2100), (7, 9)):
            u = [p - 1] * z1
            v = [p - 1] * z2
            entry = {"p": p, "z1": z1, "z2": z2, "tag": "all_p_minus_1"}
            for eng, fn in (("fft_pad", lin_conv_fft_pad), ("tft", conv_tft)):
                cnt = OpCounters()
                entry[eng] = fn(u, v, ConvRequest(fp, engine=eng, counters=cnt))
                entry[eng + "_counters"] = [cnt.butterflies, cnt.pointwise_muls]
            cases.append(entry)
    return cases


def poly_cases(rng):
    """poly_mul (normalize semantics, zero short-circuit) on DensePoly inputs."""
    out = []
    for p in (17, P2, P3):
        fp = FourierPrime.from_modulus(p)
        for u, v in (([0, 0, 0], [1, 2]), ([1, 2, 0, 0], [3, 0]), ([5], [7, 0, 0]),
                     ([p - 1, 1], [1, 1]),
                     ([rng.randrange(1, p) for _ in range(6 if p == 17 else 20)] + [0, 0],
                      [rng.randrange(1, p) for _ in range(5 if p == 17 else 9)])):
            for eng in ("fft_pad", "tft"):
                cnt = OpCounters()
                r = poly_mul(DensePoly(fp, tuple(u)), DensePoly(fp, tuple(v)),
                             ConvRequest(fp, engine=eng, counters=cnt))
                out.append({"p": p, "u": u, "v": v, "engine": eng, "out": list(r.coeffs),
                            "counters": [cnt.butterflies, cnt.pointwise_muls]})
    return out


def split_cases(rng):
    """Eq. 13 split engine (convolve.py:172-227) at several sizes and primes."""
    out = []
    for p in (17, 257, P2, P3):
        fp = FourierPrime.from_modulus(p)
        for size in (2, 4, 8, 16, 64, 256, 1024):
            if size.bit_length() - 1 > fp.two_adicity:
                continue
            u = [rng.randrange(p) for _ in range(size)]
            v = [rng.randrange(p) for _ in range(size)]
            cnt = OpCounters()
            split = circ_conv_split(u, v, ConvRequest(fp, engine="split", counters=cnt))
            a, b = split_residues(u, p)
            entry = {"p": p, "size": size, "u": u, "v": v, "split": split,
                     "split_counters": [cnt.butterflies, cnt.pointwise_muls],
                     "res_a": a, "res_b": b, "recombined": recombine_residues(a, b, p)}
            if size.bit_length() <= fp.two_adicity:  # nega_conv on `size` points needs 2*size
                cn = OpCounters()
                entry["nega"] = nega_conv(u, v, ConvRequest(fp, counters=cn))
                entry["nega_counters"] = [cn.butterflies, cn.pointwise_muls]
            out.append(entry)
    for p in (P2, P3):  # poly_mul with the split engine (normalize + counters)
        fp = FourierPrime.from_modulus(p)
        for z1, z2 in ((1, 1), (3, 7), (100, 28), (129, 1)):
            u = [rng.randrange(1, p) for _ in range(z1)]
            v = [rng.randrange(1, p) for _ in range(z2)]
            cnt = OpCounters()
            r = poly_mul(DensePoly(fp, tuple(u)), DensePoly(fp, tuple(v)),
                         ConvRequest(fp, engine="split", counters=cnt))
            out.append({"p": p, "poly": True, "u": u, "v": v, "out": list(r.coeffs),
                        "counters": [cnt.butterflies, cnt.pointwise_muls]})
    return out


def config_row(cfg, p, z1, z2, seed, rows, engine):
    """Reference poly_mul on rows of a BASELINE config (shared seeded inputs)."""
    fp = FourierPrime.from_modulus(p)
    recs = []
    for r in rows:
        a = oracle.gen_u32(seed, 0, r, 1, z1, p)[0]
        b = oracle.gen_u32(seed, 1, r, 1, z2, p)[0]
        cnt = OpCounters()
        t0 = time.perf_counter()
        res = poly_mul(DensePoly(fp, tuple(int(x) for x in a)),
                       DensePoly(fp, tuple(int(x) for x in b)),
                       ConvRequest(fp, engine=engine, counters=cnt))
        dt = time.perf_counter() - t0
        coeffs = list(res.coeffs)
        n = z1 + z2 - 1
        full = coeffs + [0] * (n - len(coeffs))
        recs.append({"row": r, "sha256": sha(full), "head": full[:8], "tail": full[-8:],
                     "normalized_len": len(coeffs),
                     "counters": [cnt.butterflies, cnt.pointwise_muls],
                     "ref_seconds": round(dt, 4)})
    return {"cfg": cfg, "p": p, "z1": z1, "z2": z2, "seed": seed, "engine": engine,
            "rows": recs}


def cfg5_pin():
    """Config 5: reference poly_mul per prime on from_ints inputs + exact CRT."""
    z = 1 << 20
    A = oracle.gen_u32(5, 0, 0, 1, z, 1 << 30)[0]
    B = oracle.gen_u32(5, 1, 0, 1, z, 1 << 30)[0]
    n = 2 * z - 1
    res = []
    per = {}
    for p in (P1, P2, P3):
        fp = FourierPrime.from_modulus(p)
        t0 = time.perf_counter()
        r = poly_mul(DensePoly.from_ints(fp, [int(x) for x in A]),
                     DensePoly.from_ints(fp, [int(x) for x in B]),
                     ConvRequest(fp, engine="fft_pad"))
        c = list(r.coeffs) + [0] * (n - len(r.coeffs))
        per[str(p)] = {"sha256": sha(c), "seconds": round(time.perf_counter() - t0, 1),
                       "head": c[:4]}
        res.append(c)
    m12 = P1 * P2
    i12 = pow(P1, -1, P2)
    i123 = pow(m12, -1, P3)
    ints = []
    for r1, r2, r3 in zip(*res):
        y2 = (r2 - r1) * i12 % P2
        x12 = r1 + P1 * y2
        y3 = (r3 - x12) * i123 % P3
        ints.append(x12 + m12 * y3)
    limbs = np.array([[x & 0xFFFFFFFF for x in ints], [(x >> 32) & 0xFFFFFFFF for x in ints],
                      [(x >> 64) & 0xFFFFFFFF for x in ints]], dtype=np.uint32)
    return {"seed": 5, "z": z, "hi": 1 << 30, "per_prime": per,
            "limbs_sha256": hashlib.sha256(limbs.tobytes()).hexdigest(),
            "max_bits": max(x.bit_length() for x in ints),
            "head": [str(x) for x in ints[:4]], "tail": [str(x) for x in ints[-4:]]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg5", action="store_true", help="also pin config 5 (~2 min)")
    ap.add_argument("--cfg4", action="store_true",
                    help="also pin config 4 rows 0 and 7 (~4 min per row)")
    args = ap.parse_args()
    rng = random.Random(0x1609_01010)
    small = {
        "generator": "tests/golden/make_golden.py",
        "reference": "modconv " + modconv.__version__ + " (/root/reference/pkg/src)",
        "fields": fields(),
        "kats": kats(),
        "transforms": transforms(rng),
        "convs": convs(rng),
        "poly_mul": poly_cases(rng),
        "split": split_cases(random.Random(0x5117)),
    }
    with open(os.path.join(HERE, "reference_small.json"), "w") as f:
        json.dump(small, f, separators=(",", ":"))
    cfgs = {
        "gen": "oracle.gen_u32(seed, stream=0 for a / 1 for b, row, 1, z, hi=p)",
        "configs": [
            config_row(1, P1, 1024, 1024, 1, [0], "fft_pad"),
            config_row(1, P1, 1024, 1024, 1, [0], "tft"),
            config_row(2, P3, 1500, 2100, 2, [0, 1, 4095], "tft"),
            config_row(2, P3, 1500, 2100, 2, [0], "fft_pad"),
            config_row(3, P2, 4096, 4096, 3, [0, 65535], "fft_pad"),
        ],
    }
    old = os.path.join(HERE, "reference_configs.json")
    prev = json.load(open(old)) if os.path.exists(old) else {}
    if args.cfg5:
        cfgs["cfg5"] = cfg5_pin()
    elif "cfg5" in prev:
        cfgs["cfg5"] = prev["cfg5"]
    if args.cfg4:
        # one reference poly_mul at L = 2^23 takes ~4 min and ~3 GB
        cfgs["cfg4"] = config_row(4, P3, 1 << 22, 1 << 22, 4, [0, 7], "fft_pad")
    elif "cfg4" in prev:
        cfgs["cfg4"] = prev["cfg4"]
    with open(os.path.join(HERE, "reference_configs.json"), "w") as f:
        json.dump(cfgs, f, indent=1)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
