"""Modular DFT and truncated transforms on the GPU, with op counting.

Mirrors the reference's transform API (/root/reference/pkg/src/modconv/
transform.py): OpCounters, TwiddleTable/get_table, moddft (natural order,
inverse scaled by 1/N), tft (first n bit-reversed spectral values), itft
(returns L*u).  The arithmetic runs in libmodconv_b200 (mc_ntt / mc_tft /
mc_itft); OpCounters are filled analytically with the reference's exact
counts (a count-only walk of the same recursions), so call-compatible
callers see identical tallies.
"""

from __future__ import annotations

import threading
from functools import lru_cache

import torch

from . import _native, _tensors
from .field import as_field, check_transform_size, root_of_unity, smallest_generator


class OpCounters:
    """Monotone tally of butterflies and pointwise products
    (transform.py:23-49)."""

    __slots__ = ("butterflies", "pointwise_muls")

    def __init__(self, butterflies: int = 0, pointwise_muls: int = 0):
        self.butterflies = butterflies
        self.pointwise_muls = pointwise_muls

    def merge(self, other) -> None:
        self.butterflies += other.butterflies
        self.pointwise_muls += other.pointwise_muls

    def __eq__(self, other) -> bool:
        if not isinstance(other, OpCounters):
            return NotImplemented
        return (self.butterflies, self.pointwise_muls) == (other.butterflies, other.pointwise_muls)

    def __repr__(self) -> str:
        return f"OpCounters(butterflies={self.butterflies}, pointwise_muls={self.pointwise_muls})"


# ------------------------------------------------------------------ counts
def full_count(L: int) -> int:
    """(L/2) log2 L butterflies of a full transform (transform.py:194-195)."""
    return (L >> 1) * (L.bit_length() - 1)


@lru_cache(maxsize=None)
def tft_count(m: int, z: int, n: int) -> int:
    """Butterflies of _tft_recurse(m, z, n) (transform.py:379-418)."""
    if n == 0 or m == 1:
        return 0
    h = m >> 1
    if n > h:
        zz = h if z > h else z
        return zz + tft_count(h, zz, h) + tft_count(h, zz, n - h)
    if z > h:
        return (z - h) + tft_count(h, h, n)
    return tft_count(h, z, n)


@lru_cache(maxsize=None)
def itft_count(m: int, n: int) -> int:
    """Butterflies of _itft_recurse(m, n) (transform.py:451-489)."""
    if m == 1 or n == 0:
        return 0
    if n == m:
        return full_count(m)
    h = m >> 1
    if n <= h:
        return (h - n) + itft_count(h, n) + n
    return itft_count(h, h) + (h - (n - h)) + itft_count(h, n - h) + (n - h)


# ------------------------------------------------------------------ tables
class TwiddleTable:
    """Host descriptor of one transform size (transform.py:52-107).

    The device tables (stage-major twiddles with Shoup quotients) live in the
    native library, cached per (device, p, size); constructing this object
    validates the size exactly like the reference and, when a GPU is present,
    prepares them.  `powers` (the L host ints of the reference) is computed
    lazily on first access only -- the GPU path never needs it.
    """

    __slots__ = ("field", "size", "log2_size", "root", "inv_size", "_powers")

    def __init__(self, field, size: int):
        fp = as_field(field)
        if size < 1 or size & (size - 1):
            raise ValueError(f"transform size must be a power of two: {size}")
        log2 = size.bit_length() - 1
        check_transform_size(fp, log2)
        self.field = fp
        self.size = size
        self.log2_size = log2
        self.root = root_of_unity(fp, size).value
        self.inv_size = pow(size, fp.p - 2, fp.p)
        self._powers = None
        if torch.cuda.is_available():
            with _generator(fp):
                _native.check(_native.lib().mc_field_prepare(fp.p, log2, -1))

    @property
    def powers(self) -> list[int]:
        if self._powers is None:
            p, w, acc, out = self.field.p, self.root, 1, []
            for _ in range(self.size):
                out.append(acc)
                acc = acc * w % p
            self._powers = out
        return self._powers

    @property
    def inv_powers(self) -> list[int]:
        pw = self.powers
        return [1] + pw[:0:-1]


_TABLE_CACHE: dict[tuple[int, int, int], TwiddleTable] = {}
_TABLE_LOCK = threading.Lock()


class _generator:
    """Run the native transforms with the field's own generator (thread-local
    selection in the library, mc_use_generator) when it is not the smallest
    primitive root -- the reference builds every table from field.generator
    (transform.py:83)."""

    __slots__ = ("p", "g")

    def __init__(self, fp):
        self.p = fp.p
        self.g = fp.generator if fp.generator != smallest_generator(fp.p) else 0

    def __enter__(self):
        if self.g:
            _native.check(_native.lib().mc_use_generator(self.p, self.g))

    def __exit__(self, *exc):
        if self.g:
            _native.lib().mc_use_generator(self.p, 0)


def get_table(field, size: int) -> TwiddleTable:
    """Shared table for (p, generator, size); built once (transform.py:110-124)."""
    fp = as_field(field)
    key = (fp.p, fp.generator, size)
    t = _TABLE_CACHE.get(key)
    if t is None:
        with _TABLE_LOCK:
            t = _TABLE_CACHE.get(key)
            if t is None:
                t = TwiddleTable(fp, size)
                _TABLE_CACHE[key] = t
    return t


# ------------------------------------------------------------------ transforms
def moddft(x, table: TwiddleTable, direction: str = "fwd", counters: OpCounters | None = None):
    """Full modular DFT, natural order in and out (transform.py:167-196)."""
    n = table.size
    if len(x) != n:
        raise ValueError(f"input length {len(x)} != table size {n}")
    if direction not in ("fwd", "inv"):
        raise ValueError(f"direction must be 'fwd' or 'inv': {direction!r}")
    dev = _tensors.require_cuda()
    p = table.field.p
    xt = _tensors.list_to_device(x, p, dev)
    y = torch.empty_like(xt)
    with _generator(table.field):
        _native.check(_native.lib().mc_ntt(_tensors.ptr(xt), _tensors.ptr(y), table.log2_size, 1,
                                           p, int(direction == "inv"), _tensors.stream_handle()))
    if counters is not None:
        counters.butterflies += full_count(n)
    return _tensors.device_to_list(y)


def moddft_naive(x, table: TwiddleTable, direction: str = "fwd"):
    """The transform's defining sum (transform.py:199-225): its output equals
    moddft's bit for bit, which is what serves it (no counters, as in the
    reference)."""
    return moddft(x, table, direction)


BASE_CASE_SIZES = (2, 4, 8)  # transform.py:222
_CODELET_COST = {2: 1, 4: 4, 8: 12}  # (m/2) log2 m, transform.py:225


def dft_basecase(x, table: TwiddleTable, direction: str = "fwd",
                 counters: OpCounters | None = None):
    """Loop-free DFT of size 2, 4 or 8 (transform.py:279-307): same output as
    moddft, same argument checks and butterfly count."""
    m = len(x)
    if m not in BASE_CASE_SIZES:
        raise ValueError(f"base case size must be one of {BASE_CASE_SIZES}: {m}")
    if table.size != m:
        raise ValueError(f"table size {table.size} != input length {m}")
    if direction not in ("fwd", "inv"):
        raise ValueError(f"direction must be 'fwd' or 'inv': {direction!r}")
    out = moddft(x, table, direction)
    if counters is not None:
        counters.butterflies += _CODELET_COST[m]
    return out


def moddft_plan(x, table: TwiddleTable, splits: tuple, base_case: int, direction: str = "fwd",
                counters: OpCounters | None = None):
    """DFT along an explicit radix decomposition (transform.py:333-376).
    Every valid plan yields moddft's output bit for bit and costs
    (N/2) log2 N butterflies; the plan is validated exactly like the
    reference, the transform runs on the GPU kernels."""
    n = table.size
    if len(x) != n:
        raise ValueError(f"input length {len(x)} != table size {n}")
    if base_case not in BASE_CASE_SIZES:
        raise ValueError(f"base case must be one of {BASE_CASE_SIZES}: {base_case}")
    prod = base_case
    for sp in splits:
        if sp not in BASE_CASE_SIZES:
            raise ValueError(f"split radix must be one of {BASE_CASE_SIZES}: {sp}")
        prod *= sp
    if prod != n:
        raise ValueError(f"decomposition {tuple(splits)} x base {base_case} != size {n}")
    if direction not in ("fwd", "inv"):
        raise ValueError(f"direction must be 'fwd' or 'inv': {direction!r}")
    out = moddft(x, table, direction)
    if counters is not None:
        counters.butterflies += full_count(n)
    return out


def tft(table: TwiddleTable, x, n: int, counters: OpCounters | None = None):
    """First n spectral values, bit-reversed order (transform.py:421-448)."""
    size = table.size
    z = len(x)
    if z < 1:
        raise ValueError("input must be nonempty")
    if z > n:
        raise ValueError(f"input length {z} exceeds output count {n}")
    if n > size:
        raise ValueError(f"output count {n} exceeds transform size {size}")
    dev = _tensors.require_cuda()
    p = table.field.p
    xt = _tensors.list_to_device(x, p, dev)
    y = torch.empty(n, dtype=torch.int32, device=dev)
    with _generator(table.field):
        _native.check(_native.lib().mc_tft(_tensors.ptr(xt), z, _tensors.ptr(y), n,
                                           table.log2_size, 1, p, _tensors.stream_handle()))
    if counters is not None:
        counters.butterflies += tft_count(size, z, n)
    return _tensors.device_to_list(y)


def itft(table: TwiddleTable, xhat, counters: OpCounters | None = None):
    """Recover L*u_i, i < n, from n bit-reversed spectral values
    (transform.py:492-529)."""
    size = table.size
    n = len(xhat)
    if n < 1:
        raise ValueError("spectral input must be nonempty")
    if n > size:
        raise ValueError(f"input length {n} exceeds transform size {size}")
    dev = _tensors.require_cuda()
    p = table.field.p
    xt = _tensors.list_to_device(xhat, p, dev)
    y = torch.empty(n, dtype=torch.int32, device=dev)
    with _generator(table.field):
        _native.check(_native.lib().mc_itft(_tensors.ptr(xt), _tensors.ptr(y), n,
                                            table.log2_size, 1, p, _tensors.stream_handle()))
    if counters is not None:
        counters.butterflies += itft_count(size, n)
    return _tensors.device_to_list(y)


def bit_reverse_permute(x: list) -> list:
    """output[rev(j)] == input[j] (transform.py:141-147); host helper."""
    n = len(x)
    if n < 1 or n & (n - 1):
        raise ValueError(f"length must be a power of two: {n}")
    bits = n.bit_length() - 1
    return [x[int(format(i, f"0{bits}b")[::-1], 2) if bits else 0] for i in range(n)]
