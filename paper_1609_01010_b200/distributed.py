"""Multi-GPU plumbing for the modular-convolution path (one process per GPU,
torch.distributed over NCCL; gloo for CPU tests).

The path shards without exchange: independent products of a batch are
partitioned by contiguous row ranges (configs 2-4), and the three primes of
the integer product (config 5) are spread over ranks.  The only collective
is the gather of config 5's residue vectors onto the rank that runs the CRT
kernel.  Nothing here is on the reference's side:
the reference has no distributed component.
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from .crt import PRIMES


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def shard_rows(batch: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [row0, row0 + rows) of `batch` rows for `rank`
    (sizes differ by at most one)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad world size / rank")
    base, extra = divmod(batch, world_size)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


def primes_of_rank(world_size: int, rank: int) -> list[int]:
    """Prime indices (into PRIMES) computed by `rank`: round-robin, so at
    world size >= 3 ranks 0, 1, 2 own one prime each."""
    return [k for k in range(3) if k % world_size == rank]


def _gpu_prime_product(a: torch.Tensor, b: torch.Tensor, k: int) -> torch.Tensor:
    from . import _native, _tensors

    n = a.numel() + b.numel() - 1
    r = torch.empty(n, dtype=torch.int32, device=a.device)
    _native.check(_native.lib().mc_mul_mod_prime_k(a.data_ptr(), a.numel(), b.data_ptr(),
                                                    b.numel(), r.data_ptr(), k,
                                                    _tensors.stream_handle()))
    return r


def _gpu_crt(r1, r2, r3) -> torch.Tensor:
    from .crt import crt3

    return crt3(r1, r2, r3)


def mul_three_primes_distributed(a: torch.Tensor, b: torch.Tensor, dst: int = 0, group=None,
                                 prime_product: Callable | None = None,
                                 crt: Callable | None = None):
    """Exact integer product of a and b (int32 words, identical on every
    rank), primes spread over the ranks of `group`.

    Each rank computes the residue vectors of its primes; rank `dst`
    gathers all three (torch.distributed.gather: send/recv over NCCL) and
    runs the Garner CRT kernel.  Returns the limbs [3, n] on `dst`, None
    elsewhere.  `prime_product(a, b, k)` and `crt(r1, r2, r3)` default to
    the GPU kernels; tests inject CPU checkers to exercise the
    orchestration under gloo.
    """
    prime_product = prime_product or _gpu_prime_product
    crt = crt or _gpu_crt
    ws = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = a.numel() + b.numel() - 1
    mine = {k: prime_product(a, b, k) for k in primes_of_rank(ws, rank)}
    if ws == 1:
        return crt(mine[0], mine[1], mine[2])
    # one gather per prime from its owner (ranks >= 3 own nothing); under a
    # host backend (gloo) device tensors travel through host memory
    host_coll = dist.get_backend(group) != "nccl" and a.device.type == "cuda"
    residues = {}
    for k in range(3):
        owner = k % ws
        if owner == dst:
            if rank == dst:
                residues[k] = mine[k]
            continue
        if rank == owner:
            t = mine[k].contiguous()
            dist.send(t.cpu() if host_coll else t, dst=dst, group=group)
        elif rank == dst:
            buf = torch.empty(n, dtype=torch.int32, device="cpu" if host_coll else a.device)
            dist.recv(buf, src=owner, group=group)
            residues[k] = buf.to(a.device) if host_coll else buf
    if rank != dst:
        return None
    return crt(residues[0], residues[1], residues[2])
