"""Golden transforms for fields whose generator is NOT the smallest primitive
root, produced by the unmodified reference (/root/reference/pkg/src): its
TwiddleTable takes w_L = generator^((p-1)/L) from the FourierPrime it is
given (transform.py:83, field.py:209-224).

    python tests/golden/make_golden_generators.py   # -> reference_generators.json
"""

from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from modconv import FourierPrime, OpCounters, itft, moddft, tft  # noqa: E402
from modconv.transform import TwiddleTable  # noqa: E402


def other_generator(p: int, skip: int) -> int:
    """The (skip+1)-th primitive root above the smallest one."""
    fp = FourierPrime.from_modulus(p)
    g = fp.generator + 1
    while True:
        try:
            FourierPrime(p, fp.two_adicity, g)
            if skip == 0:
                return g
            skip -= 1
        except ValueError:
            pass
        g += 1


def main():
    rng = random.Random(0x6E11)
    cases = []
    for p, skip, sizes in ((17, 0, (2, 4, 8, 16)), (257, 3, (16, 64, 256)),
                           (2013265921, 0, (16, 1024, 4096, 1 << 14)),
                           (469762049, 1, (64, 2048)), (998244353, 2, (8192,))):
        g = other_generator(p, skip)
        fp = FourierPrime(p, FourierPrime.from_modulus(p).two_adicity, g)
        for L in sizes:
            t = TwiddleTable(fp, L)  # direct: get_table caches per (p, L) only
            x = [rng.randrange(p) for _ in range(L)]
            n = max(1, L - L // 3)
            z = max(1, n // 2)
            xs = x[:z]
            c1, c2 = OpCounters(), OpCounters()
            y = tft(t, xs, n, c1)
            cases.append({"p": p, "g": g, "L": L, "root": t.root, "x": x,
                          "fwd": moddft(x, t, "fwd"), "inv": moddft(x, t, "inv"),
                          "tft_in": xs, "n": n, "tft_out": y,
                          "itft_out": itft(t, y, c2),
                          "counters": [c1.butterflies, c2.butterflies]})
    with open(os.path.join(HERE, "reference_generators.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden_generators.py", "cases": cases}, f,
                  separators=(",", ":"))
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
