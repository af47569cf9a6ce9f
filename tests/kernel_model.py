"""Pure-Python model of the fused small-L convolution kernel's schedule.

Test helper (CPU): mirrors, stage by stage, what
paper_1609_01010_b200/csrc/conv_small.cu computes, so the pruning rules of
the relaxed truncated transforms can be checked against the oracle without a
GPU.  Position-level (not thread-level): the kernel groups these stages into
register passes; the arithmetic and the set of butterflies executed are the
same.

  * forward: decimation-in-frequency, natural in -> bit-reversed out, direct
    per-stage twiddles Tf[h + j] = w_{2h}^j (w the reference root,
    transform.py:84-107);
  * relaxed TFT: outputs are computed for the first n' = N*G positions
    (G = L / R_top, N = ceil(n / G)); stages with half-size h >= G skip
    butterflies whose outputs are not needed and exploit known-zero inputs
    (same rules as transform.py:379-418);
  * inverse: complete inverse DIT on each active G-block first, then the
    van der Hoeven recursion (transform.py:451-489) over the top levels with
    base case m == G.
"""

from __future__ import annotations


def tables(p: int, L: int, w: int):
    """Tf[h + j] = w_{2h}^j, Ti[h + j] = w_{2h}^{-j} for 1 <= h < L, j < h."""
    Tf = [0] * max(L, 1)
    Ti = [0] * max(L, 1)
    h = 1
    while h < L:
        w2h = pow(w, L // (2 * h), p)
        inv = pow(w2h, p - 2, p)
        for j in range(h):
            Tf[h + j] = pow(w2h, j, p)
            Ti[h + j] = pow(inv, j, p)
        h <<= 1
    return Tf, Ti


def r_top(L: int) -> int:
    return min(16, L)


def fwd_tft_relaxed(x, z: int, N: int, L: int, p: int, Tf):
    """Relaxed truncated DIF.  Returns (values[L], butterflies_executed)."""
    G = L // r_top(L)
    nn = N * G
    c = list(x) + [0] * (L - len(x))
    for i in range(z, L):
        c[i] = 0
    count = 0
    h = L >> 1
    while h >= 1:
        for x0 in range(L):
            if x0 & h:
                continue
            b = x0 - (x0 % (2 * h))
            if b >= nn:
                continue
            j = x0 % (2 * h)
            if h >= G:
                a_zero = j >= z
                b_zero = j + h >= z
                hi_needed = b + h < nn
            else:
                a_zero = b_zero = False
                hi_needed = True
            if a_zero:
                continue
            a, bb = c[x0], c[x0 + h]
            w = Tf[h + j]
            if hi_needed:
                if b_zero:
                    c[x0 + h] = a * w % p
                else:
                    c[x0] = (a + bb) % p
                    c[x0 + h] = (a - bb) * w % p
                count += 1
            else:
                if not b_zero:
                    c[x0] = (a + bb) % p
                    count += 1
        h >>= 1
    return c, count


def inv_tft_relaxed(c, N: int, L: int, p: int, Tf, Ti):
    """Relaxed inverse: c[:N*G] spectral (bit-reversed), c[N*G:] time values
    (zero for a product).  Returns L * u in c[:N*G] (in place) and the
    butterfly count."""
    G = L // r_top(L)
    count = 0
    # 1. complete inverse DIT on active G-blocks (stages h < G)
    for blk in range(N):
        off = blk * G
        h = 1
        while h < G:
            for x0 in range(off, off + G):
                if x0 & h:
                    continue
                j = x0 % h
                t = c[x0 + h] * Ti[h + j] % p
                a = c[x0]
                c[x0] = (a + t) % p
                c[x0 + h] = (a - t) % p
                count += 1
            h <<= 1

    pow2 = {}

    def m_mod(m):
        return m % p

    def rec(off, m, n):
        nonlocal count
        if m == G or n == 0:
            return
        h = m >> 1
        if n <= h:
            for j in range(n, h):
                c[off + j] = (c[off + j] + c[off + j + h]) % p
                count += 1
            rec(off, h, n)
            mm = m_mod(m)
            for i in range(n):
                c[off + i] = (2 * c[off + i] - mm * c[off + i + h]) % p
                count += 1
            return
        rec(off, h, h)
        mm = m_mod(m)
        inv_h = pow(h, p - 2, p)
        for i in range(n - h, h):
            lo, hi = off + i, off + i + h
            a, b = c[lo], c[hi]
            c[hi] = (a * inv_h - 2 * b) % p * Tf[h + i] % p
            c[lo] = (2 * a - mm * b) % p
            count += 1
        rec(off + h, h, n - h)
        for i in range(n - h):
            lo, hi = off + i, off + i + h
            t = c[hi] * Ti[h + i] % p
            a = c[lo]
            c[lo] = (a + t) % p
            c[hi] = (a - t) % p
            count += 1

    rec(0, L, N * G)
    del pow2
    return c, count


def conv_tft_model(u, v, p: int, w_of_L):
    """Full relaxed-TFT product as the kernel computes it."""
    z1, z2 = len(u), len(v)
    n = z1 + z2 - 1
    L = 1
    while L < n:
        L <<= 1
    R = r_top(L)
    G = L // R
    N = -(-n // G)
    Tf, Ti = tables(p, L, w_of_L(L))
    fa, c1 = fwd_tft_relaxed(u, z1, N, L, p, Tf)
    fb, c2 = fwd_tft_relaxed(v, z2, N, L, p, Tf)
    Linv = pow(L, p - 2, p)
    prod = [fa[i] * fb[i] % p * Linv % p if i < N * G else 0 for i in range(L)]
    out, c3 = inv_tft_relaxed(prod, N, L, p, Tf, Ti)
    return out[:n], (c1, c2, c3)
