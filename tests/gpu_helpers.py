"""Helpers shared by the GPU parity tests (input generation on device,
evaluation-homomorphism checker)."""

from __future__ import annotations

import hashlib

import numpy as np
import torch

from paper_1609_01010_b200 import _native, _tensors


def gen_device(seed: int, stream: int, row0: int, rows: int, length: int, hi: int,
               ld: int | None = None) -> torch.Tensor:
    """Seeded inputs generated on the GPU (same generator as oracle.gen_u32)."""
    ld = ld or length
    t = torch.empty((rows, ld), dtype=torch.int32, device="cuda")
    _native.check(_native.lib().mc_gen_u32(seed, stream, row0, rows, length, hi, t.data_ptr(),
                                           ld, _tensors.stream_handle()))
    return t[:, :length] if ld != length else t


def to_u32_np(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def sha_row(row: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(row, dtype=np.uint32).tobytes()).hexdigest()


def eval_rows_gpu(c: torch.Tensor, x: torch.Tensor, p: int) -> torch.Tensor:
    """Horner evaluation of every row of c (int32 residues) at x (int64 [B])
    mod p, in int64 on the GPU (values < 2^31 so products < 2^62)."""
    acc = torch.zeros(c.shape[0], dtype=torch.int64, device=c.device)
    cc = c.to(torch.int64) & 0xFFFFFFFF
    for j in range(c.shape[1] - 1, -1, -1):
        acc = (acc * x + cc[:, j]) % p
    return acc


def eval_check(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, p: int, seed: int = 99,
               chunk: int = 16384) -> None:
    """eval(c, x) == eval(a, x) * eval(b, x) mod p at 2 seeded points per row
    (poly.py:172-181; the reference's own homomorphism property,
    tests/test_poly.py:130-135).  False-pass probability <= (n/p)^2 per row."""
    g = torch.Generator().manual_seed(seed)
    B = a.shape[0]
    for r0 in range(0, B, chunk):
        r1 = min(B, r0 + chunk)
        for _ in range(2):
            x = torch.randint(1, p, (r1 - r0,), generator=g, dtype=torch.int64).cuda()
            lhs = eval_rows_gpu(c[r0:r1], x, p)
            rhs = eval_rows_gpu(a[r0:r1], x, p) * eval_rows_gpu(b[r0:r1], x, p) % p
            bad = torch.nonzero(lhs != rhs).flatten()
            assert bad.numel() == 0, f"eval mismatch at rows {(bad[:8] + r0).tolist()}"


def powmod_vec(x: torch.Tensor, e: torch.Tensor, p: int) -> torch.Tensor:
    """x^e mod p elementwise (int64, x < p < 2^31), by square-and-multiply."""
    r = torch.ones_like(e)
    b = x.expand_as(e).clone() % p
    e = e.clone()
    while bool((e > 0).any()):
        odd = (e & 1) == 1
        r = torch.where(odd, r * b % p, r)
        b = b * b % p
        e = e >> 1
    return r


def eval_vec(c: torch.Tensor, x: int, p: int, chunk: int = 1 << 22) -> int:
    """c(x) mod p for one long residue vector (int32/uint32 on the GPU)."""
    n = c.numel()
    acc = 0
    xt = torch.tensor([x], dtype=torch.int64, device=c.device)
    for i0 in range(0, n, chunk):
        i1 = min(n, i0 + chunk)
        idx = torch.arange(i0, i1, dtype=torch.int64, device=c.device)
        w = powmod_vec(xt, idx, p)
        v = (c.reshape(-1)[i0:i1].to(torch.int64) & 0xFFFFFFFF) % p
        acc = (acc + int(((v * w) % p).sum().item())) % p
    return acc
