"""ctypes front-end of the C restatement of the reference path.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as
the checker) and bench.py's cpu_baseline / --impl reference legs.  The product
package never imports it.

Reference being restated: /root/reference/pkg/src/modconv (pure Python);
see oracle/modconv_oracle.c for the per-function file:line citations.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libmodconv_oracle.so")
_lib = None

ENGINE_FFT_PAD = 0
ENGINE_TFT = 1

u32p = ctypes.POINTER(ctypes.c_uint32)
i64p = ctypes.POINTER(ctypes.c_int64)


def build() -> str:
    """Compile the oracle library (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_gen_u32.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                  u32p, ctypes.c_int64]
        L.orc_gen_u32.restype = None
        L.orc_gen_key.argtypes = [ctypes.c_uint64] * 3
        L.orc_gen_key.restype = ctypes.c_uint64
        L.orc_primitive_root.argtypes = [ctypes.c_uint64]
        L.orc_primitive_root.restype = ctypes.c_uint64
        L.orc_two_adicity.argtypes = [ctypes.c_uint64]
        L.orc_two_adicity.restype = ctypes.c_int
        L.orc_root_of_unity.argtypes = [ctypes.c_uint64, ctypes.c_int]
        L.orc_root_of_unity.restype = ctypes.c_uint64
        L.orc_moddft.argtypes = [ctypes.c_uint32, ctypes.c_int, u32p, u32p, ctypes.c_int]
        L.orc_moddft.restype = ctypes.c_int64
        L.orc_tft.argtypes = [ctypes.c_uint32, ctypes.c_int, u32p, ctypes.c_int64, u32p,
                              ctypes.c_int64]
        L.orc_tft.restype = ctypes.c_int64
        L.orc_itft.argtypes = [ctypes.c_uint32, ctypes.c_int, u32p, ctypes.c_int64, u32p]
        L.orc_itft.restype = ctypes.c_int64
        L.orc_conv_batch.argtypes = [ctypes.c_uint32, ctypes.c_int, u32p, ctypes.c_int64,
                                     ctypes.c_int64, u32p, ctypes.c_int64, ctypes.c_int64,
                                     u32p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, i64p]
        L.orc_conv_batch.restype = ctypes.c_int
        L.orc_crt3.argtypes = [ctypes.c_uint32] * 3 + [u32p] * 3 + [ctypes.c_int64, u32p]
        L.orc_crt3.restype = None
        L.orc_mul_three_primes.argtypes = [u32p, ctypes.c_int64, u32p, ctypes.c_int64, u32p,
                                           ctypes.c_int]
        L.orc_mul_three_primes.restype = ctypes.c_int
        L.orc_tft_count.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64]
        L.orc_tft_count.restype = ctypes.c_int64
        L.orc_itft_count.argtypes = [ctypes.c_int, ctypes.c_int64]
        L.orc_itft_count.restype = ctypes.c_int64
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(u32p)


def _u32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64).astype(np.uint32))


class OracleError(ValueError):
    pass


class OracleUnsupportedSize(OracleError):
    pass


def _check(rc):
    if rc == -1:
        raise OracleUnsupportedSize("transform size exceeds the field's 2-adicity")
    if rc == -2:
        raise OracleError("usage error")
    return rc


# ---------------------------------------------------------------- generator
def gen_u32(seed: int, stream: int, row0: int, rows: int, length: int, hi: int) -> np.ndarray:
    """Seeded uniform [0, hi) words; row r of the result is row (row0 + r).

    Same definition as oracle/modconv_oracle.c orc_gen_u32 and the CUDA
    generator in the product package (bench/test input builder).
    """
    out = np.empty((rows, length), dtype=np.uint32)
    if rows and length:
        lib().orc_gen_u32(seed, stream, row0, rows, length, hi, _ptr(out), length)
    return out


# ---------------------------------------------------------------- field
def primitive_root(p: int) -> int:
    return int(lib().orc_primitive_root(p))


def two_adicity(p: int) -> int:
    return int(lib().orc_two_adicity(p))


def root_of_unity(p: int, log2n: int) -> int:
    return int(lib().orc_root_of_unity(p, log2n))


# ---------------------------------------------------------------- transforms
def moddft(x, p: int, inverse: bool = False):
    x = _u32(x)
    L = x.size
    lg = L.bit_length() - 1
    if L < 1 or L & (L - 1):
        raise OracleError("length must be a power of two")
    y = np.empty_like(x)
    bf = _check(lib().orc_moddft(p, lg, _ptr(x), _ptr(y), int(inverse)))
    return y, bf


def tft(x, n: int, L: int, p: int):
    x = _u32(x)
    y = np.empty(n, dtype=np.uint32)
    bf = _check(lib().orc_tft(p, L.bit_length() - 1, _ptr(x), x.size, _ptr(y), n))
    return y, bf


def itft(xhat, L: int, p: int):
    xhat = _u32(xhat)
    n = xhat.size
    y = np.empty(n, dtype=np.uint32)
    bf = _check(lib().orc_itft(p, L.bit_length() - 1, _ptr(xhat), n, _ptr(y)))
    return y, bf


def conv_batch(a: np.ndarray, b: np.ndarray, p: int, engine: int = ENGINE_FFT_PAD,
               threads: int = 1):
    """Row-wise linear convolutions mod p.  a: [B, z1], b: [B, z2] -> [B, n].

    Returns (c, butterflies, pointwise_muls) with reference OpCounters
    semantics (engine functions: convolve.py:160-169 / :230-253).
    """
    a = np.ascontiguousarray(np.atleast_2d(a), dtype=np.uint32)
    b = np.ascontiguousarray(np.atleast_2d(b), dtype=np.uint32)
    B, z1 = a.shape
    z2 = b.shape[1]
    n = z1 + z2 - 1
    c = np.empty((B, n), dtype=np.uint32)
    counters = (ctypes.c_int64 * 2)(0, 0)
    _check(lib().orc_conv_batch(p, engine, _ptr(a), z1, z1, _ptr(b), z2, z2, _ptr(c), n, B,
                                threads, counters))
    return c, counters[0], counters[1]


def crt3(r1, r2, r3, primes=(469762049, 998244353, 2013265921)) -> np.ndarray:
    r1, r2, r3 = _u32(r1), _u32(r2), _u32(r3)
    n = r1.size
    limbs = np.empty((3, n), dtype=np.uint32)
    lib().orc_crt3(primes[0], primes[1], primes[2], _ptr(r1), _ptr(r2), _ptr(r3), n,
                   _ptr(limbs))
    return limbs


def mul_three_primes(a, b, threads: int = 1) -> np.ndarray:
    a, b = _u32(a), _u32(b)
    n = a.size + b.size - 1
    limbs = np.empty((3, n), dtype=np.uint32)
    _check(lib().orc_mul_three_primes(_ptr(a), a.size, _ptr(b), b.size, _ptr(limbs), threads))
    return limbs


def limbs_to_ints(limbs: np.ndarray) -> list[int]:
    l0, l1, l2 = (limbs[i].astype(object) for i in range(3))
    return [int(x) | (int(y) << 32) | (int(z) << 64) for x, y, z in zip(l0, l1, l2)]


def tft_count(L: int, z: int, n: int) -> int:
    return int(lib().orc_tft_count(L.bit_length() - 1, z, n))


def itft_count(L: int, n: int) -> int:
    return int(lib().orc_itft_count(L.bit_length() - 1, n))


def schoolbook(u, v, p: int) -> list[int]:
    """Quadratic product (poly.py:90-97), pure Python: small cases only."""
    res = [0] * (len(u) + len(v) - 1)
    for i, ui in enumerate(u):
        if ui:
            for j, vj in enumerate(v):
                res[i + j] += int(ui) * int(vj)
    return [r % p for r in res]


def eval_mod(c: np.ndarray, x: np.ndarray, p: int) -> np.ndarray:
    """Row-wise polynomial evaluation c_r(x_r) mod p (Horner in blocks, int64).

    Used for the evaluation-homomorphism check (poly.py:172-181 semantics).
    c: [B, n] residues, x: [B] points.  Exact: every product is < 2^62.
    """
    c = np.atleast_2d(c).astype(np.uint64)
    x = np.asarray(x, dtype=np.uint64).reshape(-1, 1)
    p64 = np.uint64(p)
    acc = np.zeros((c.shape[0], 1), dtype=np.uint64)
    for j in range(c.shape[1] - 1, -1, -1):
        acc = (acc * x + c[:, j:j + 1]) % p64
    return acc[:, 0]
