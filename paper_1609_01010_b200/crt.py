"""Three-primes integer polynomial product over Z (config 5).

No reference counterpart: the reference lists "three-primes integer
multiplication" as out of its scope.  This is the API the
build defines for it:

  mul_three_primes(a, b) -> list[int]          exact coefficients over Z
  mul_three_primes_tensor(a, b) -> [3, n]      planar little-endian limbs

Inputs are non-negative integers < 2^32; each is reduced mod
p1 = 469762049, p2 = 998244353, p3 = 2013265921 on the fly (the
DensePoly.from_ints semantics, poly.py:46-49), the three products run through
the fft_pad engine, and a Garner CRT kernel writes x < p1*p2*p3 (~2^89.6) as
3 x 32-bit limbs.  Exact while min(z1, z2) * max(a) * max(b) < p1*p2*p3
(config 5: 2^20 * (2^30)^2 < 2^80).
"""

from __future__ import annotations

import torch

from . import _native, _tensors

PRIMES = (469762049, 998244353, 2013265921)
MODULUS = PRIMES[0] * PRIMES[1] * PRIMES[2]


def _dev_words(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = _tensors.as_words(x.reshape(-1))
        # page-locked host rows: a stream-ordered copy, so the host goes on to
        # enqueue the transforms while the copy engine runs
        return t.to(device, non_blocking=t.device.type == "cpu" and t.is_pinned()).contiguous()
    vals = [int(v) for v in x]
    if any(v < 0 or v >= (1 << 32) for v in vals):
        raise ValueError("three-primes inputs must be integers in [0, 2^32)")
    return torch.tensor(vals, dtype=torch.int64).to(torch.int32 if max(vals, default=0) < 2**31
                                                     else torch.int64).to(device).to(torch.int32)


def mul_three_primes_tensor(a, b, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Exact product limbs [3, n] (int32 bit patterns of uint32 limbs)."""
    if stream is not None and stream != torch.cuda.current_stream():
        # temporaries, scratch and the H2D copies then belong to `stream`
        with torch.cuda.stream(stream):
            return mul_three_primes_tensor(a, b, out, None)
    dev = _tensors.require_cuda()
    a_d = _dev_words(a, dev)
    b_d = _dev_words(b, dev)
    z1, z2 = a_d.numel(), b_d.numel()
    if z1 < 1 or z2 < 1:
        raise ValueError("inputs must be nonempty")
    n = z1 + z2 - 1
    if out is None:
        out = torch.empty((3, n), dtype=torch.int32, device=dev)
    elif out.shape != (3, n) or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous [3, {n}] tensor")
    words = int(_native.lib().mc_three_primes_scratch_words(z1, z2))
    scratch = torch.empty(max(words, 1), dtype=torch.int32, device=dev)
    _native.check(_native.lib().mc_mul_three_primes(
        _tensors.ptr(a_d), z1, _tensors.ptr(b_d), z2, _tensors.ptr(out), _tensors.ptr(scratch),
        _tensors.stream_handle(stream)))
    return out


def limbs_to_ints(limbs: torch.Tensor) -> list[int]:
    l = (limbs.to("cpu").to(torch.int64) & 0xFFFFFFFF).tolist()
    return [x | (y << 32) | (z << 64) for x, y, z in zip(l[0], l[1], l[2])]


def mul_three_primes(a, b) -> list[int]:
    """Exact integer coefficients of a*b (a, b: sequences of ints in [0, 2^32))."""
    return limbs_to_ints(mul_three_primes_tensor(a, b))


def crt3(r1: torch.Tensor, r2: torch.Tensor, r3: torch.Tensor, out=None,
         stream=None) -> torch.Tensor:
    """Garner CRT of residue vectors mod PRIMES -> limbs [3, n]."""
    if stream is not None and stream != torch.cuda.current_stream():
        with torch.cuda.stream(stream):
            return crt3(r1, r2, r3, out, None)
    r1, r2, r3 = (_tensors.as_words(r.reshape(-1)).contiguous() for r in (r1, r2, r3))
    n = r1.numel()
    if r2.numel() != n or r3.numel() != n:
        raise ValueError("residue vectors must have equal length")
    if out is None:
        out = torch.empty((3, n), dtype=torch.int32, device=r1.device)
    _native.check(_native.lib().mc_crt3(_tensors.ptr(r1), _tensors.ptr(r2), _tensors.ptr(r3),
                                        _tensors.ptr(out), n, _tensors.stream_handle(stream)))
    return out
