"""Multi-GPU plumbing for the modular-convolution path (one process per GPU,
torch.distributed over NCCL; gloo for CPU tests).

The path shards without exchange: independent products of a batch are
partitioned by contiguous row ranges (configs 2-4), and the three primes of
the integer product (config 5) are spread over ranks.  The only exchange is
config 5's residue vectors meeting in the CRT, done
two ways:

* mul_three_primes_p2p (default on GPUs): each rank's Garner kernel reads
  the residue vectors from the GPUs that computed them and writes its slice
  of the limbs into the destination rank's buffer, all over NVLink peer
  memory (CUDA IPC) -- the gather fused into the CRT kernel; the process
  group only carries the IPC handles and two barriers;
* mul_three_primes_distributed: residues sent to the CRT rank with
  torch.distributed send/recv (NCCL), then one CRT kernel there.

Nothing here is on the reference's side: the reference has no distributed
component.
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


# ---------------------------------------------------------------- peer memory
class _PeerCrt:
    """IPC-shared buffers of the fused distributed CRT for one (n, dst,
    group): every rank owns a [3][n] residue buffer (it writes the planes of
    its primes), dst owns the [3][n] limb buffer; every rank maps all of
    them.  Cached per shape: opening IPC handles costs milliseconds."""

    def __init__(self, n: int, dst: int, group):
        import ctypes

        from . import _native

        self.lib = _native.lib()
        self.ws = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = n
        self._own, self._opened = [], []
        res, h_res = self._alloc(12 * n)
        out, h_out = (self._alloc(12 * n) if self.rank == dst else (None, None))
        handles = [None] * self.ws
        dist.all_gather_object(handles, (h_res, h_out), group=group)
        self.res = [res if r == self.rank else self._open(handles[r][0]) for r in range(self.ws)]
        self.out = out if self.rank == dst else self._open(handles[dst][1])
        self._ctypes = ctypes

    def _alloc(self, nbytes):
        import ctypes

        from . import _native

        ptr = ctypes.c_void_p()
        h = ctypes.create_string_buffer(64)
        _native.check(self.lib.mc_ipc_alloc(nbytes, ctypes.byref(ptr), h))
        self._own.append(ptr.value)
        return ptr.value, h.raw

    def _open(self, handle):
        import ctypes

        from . import _native

        ptr = ctypes.c_void_p()
        _native.check(self.lib.mc_ipc_open(handle, ctypes.byref(ptr)))
        self._opened.append(ptr.value)
        return ptr.value

    def close(self):
        for p in self._opened:
            self.lib.mc_ipc_close(p)
        for p in self._own:
            self.lib.mc_ipc_free(p)
        self._opened, self._own = [], []


_PEER_CACHE: dict = {}


def close_peer_buffers(group=None) -> None:
    """Release the cached IPC buffers (collective: call on every rank)."""
    if dist.is_initialized():
        dist.barrier(group=group)
    for st in _PEER_CACHE.values():
        st.close()
    _PEER_CACHE.clear()


def _stream_barrier(group, device) -> None:
    """Barrier ordered on the current CUDA stream.

    Under NCCL: a one-word all-reduce.  Its kernel on every rank starts only
    after the work already queued on that rank's stream and ends only when
    every rank has contributed, and the caller's stream waits on it on the
    device -- so after it, every rank's earlier kernels are done, with no
    host synchronization and no host round trip.  Under a host backend
    (gloo: CPU tests, one shared GPU) the host synchronizes its stream and
    meets the others in dist.barrier."""
    if dist.get_backend(group) == "nccl":
        flag = _BARRIER_WORDS.get(device)
        if flag is None:
            flag = _BARRIER_WORDS[device] = torch.zeros(1, dtype=torch.int32, device=device)
        dist.all_reduce(flag, group=group)
    else:
        if device.type == "cuda":
            torch.cuda.current_stream(device).synchronize()
        dist.barrier(group=group)


_BARRIER_WORDS: dict = {}


def mul_three_primes_p2p(a: torch.Tensor, b: torch.Tensor, dst: int = 0, group=None):
    """Exact integer product of a and b (int32 words on this rank's GPU,
    identical on every rank), primes spread over the ranks; the residue
    gather is fused into the CRT kernel over peer memory.

    Rank r computes the residue planes of its primes (k % ws == r) into its
    IPC-shared buffer; after a barrier every rank runs the Garner kernel on
    its coefficient slice (shard_rows(n, ws, r)), loading the three residue
    planes from their owners' GPUs and storing its limbs straight into
    dst's buffer over NVLink; after a second barrier dst copies the limbs
    out.  Under NCCL both barriers are stream-ordered one-word all-reduces
    (_stream_barrier): the call enqueues everything and returns without a
    host synchronization.  Returns [3, n] int32 limbs on dst, None
    elsewhere.
    """
    from . import _native, _tensors

    ws = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if ws == 1:
        from .crt import mul_three_primes_tensor

        return mul_three_primes_tensor(a, b)
    lib = _native.lib()
    z1, z2 = a.numel(), b.numel()
    n = z1 + z2 - 1
    key = (n, dst, id(group), ws)
    st = _PEER_CACHE.get(key)
    if st is None:
        st = _PEER_CACHE[key] = _PeerCrt(n, dst, group)
    stream = _tensors.stream_handle()
    a_, b_ = a.contiguous(), b.contiguous()
    for k in primes_of_rank(ws, rank):
        _native.check(lib.mc_mul_mod_prime_k(a_.data_ptr(), z1, b_.data_ptr(), z2,
                                             st.res[rank] + 4 * k * n, k, stream))
    _stream_barrier(group, a.device)  # every residue plane is written
    lo, cnt = shard_rows(n, ws, rank)
    r = [st.res[k % ws] + 4 * (k * n + lo) for k in range(3)]
    _native.check(lib.mc_crt3_slice(r[0], r[1], r[2], st.out + 4 * lo, n, cnt, stream))
    # every limb slice is in dst's buffer, and no rank reads a residue plane
    # any more (the next call may overwrite them)
    _stream_barrier(group, a.device)
    if rank != dst:
        return None
    out = torch.empty((3, n), dtype=torch.int32, device=a.device)
    _native.check(lib.mc_copy_device(out.data_ptr(), st.out, 12 * n, stream))
    return out
