"""Fused distributed CRT (mul_three_primes_p2p) on the one GPU of the box:
2 and 3 processes share cuda:0, exchange CUDA IPC handles over a gloo
process group, compute their primes' residue planes, and run one Garner
slice each that reads the planes from the other processes' buffers and
writes its limbs into rank 0's buffer.  The kernels never wait on one
another (host barriers only), so sharing one device is sound; on a multi-GPU
node the same loads and stores cross NVLink."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(z1, z2):
    rng = np.random.default_rng(7 + z1)
    a = rng.integers(0, 1 << 30, z1, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 1 << 30, z2, dtype=np.uint64).astype(np.uint32)
    a[:3] = (1 << 30) - 1
    b[-3:] = (1 << 30) - 1
    return a, b


def _worker(rank, ws, port, out_dir, sizes):
    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_1609_01010_b200.distributed import close_peer_buffers, mul_three_primes_p2p

    for z1, z2 in sizes:
        a_np, b_np = _inputs(z1, z2)
        a = torch.from_numpy(a_np.view(np.int32)).cuda()
        b = torch.from_numpy(b_np.view(np.int32)).cuda()
        for rep in range(2):  # the second call reuses the cached peer buffers
            res = mul_three_primes_p2p(a, b, dst=0)
            if rank == 0:
                np.save(os.path.join(out_dir, f"limbs_{z1}_{z2}_{rep}.npy"),
                        res.cpu().numpy().view(np.uint32))
            else:
                assert res is None
    close_peer_buffers()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_three_primes_p2p_crt(tmp_path, orc, ws):
    sizes = [(3000, 2000), (9000, 7001)]  # fused kernel, four-step (L = 2^14)
    mp.spawn(_worker, args=(ws, _free_port(), str(tmp_path), sizes), nprocs=ws, join=True)
    for z1, z2 in sizes:
        a, b = _inputs(z1, z2)
        want = orc.mul_three_primes(a, b)
        for rep in range(2):
            assert np.array_equal(np.load(tmp_path / f"limbs_{z1}_{z2}_{rep}.npy"), want), (z1, z2, rep)


def test_crt3_slice_matches_full(orc):
    """Slices with the full-length limb stride tile mc_crt3 exactly."""
    import paper_1609_01010_b200 as mc
    from paper_1609_01010_b200 import _native

    n = 100_003
    rng = np.random.default_rng(5)
    rs = [torch.from_numpy(rng.integers(0, p, n, dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
          for p in mc.PRIMES]
    full = mc.crt3(*rs)
    out = torch.full((3, n), -1, dtype=torch.int32, device="cuda")
    lib = _native.lib()
    st = torch.cuda.current_stream().cuda_stream
    for lo, cnt in ((0, 40_000), (40_000, 1), (40_001, 60_002)):
        _native.check(lib.mc_crt3_slice(rs[0].data_ptr() + 4 * lo, rs[1].data_ptr() + 4 * lo,
                                        rs[2].data_ptr() + 4 * lo, out.data_ptr() + 4 * lo, n,
                                        cnt, st))
    torch.cuda.synchronize()
    assert torch.equal(out, full)


def _nccl_worker(rank, port, out_dir):
    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=1, device_id=torch.device("cuda:0"))
    from paper_1609_01010_b200 import distributed as D

    assert dist.get_backend() == "nccl"
    a_np, b_np = _inputs(9000, 7001)
    a = torch.from_numpy(a_np.view(np.int32)).cuda()
    b = torch.from_numpy(b_np.view(np.int32)).cuda()
    # the stream-ordered barrier is a one-word NCCL all-reduce queued behind
    # the product kernels; the limbs copied after it must be complete
    r = D.mul_three_primes_distributed(a, b, dst=0)
    D._stream_barrier(None, a.device)
    np.save(os.path.join(out_dir, "nccl_dist.npy"), r.cpu().numpy().view(np.uint32))
    r = D.mul_three_primes_p2p(a, b, dst=0)
    np.save(os.path.join(out_dir, "nccl_p2p.npy"), r.cpu().numpy().view(np.uint32))
    dist.destroy_process_group()


def test_nccl_process_group_world_size_1(tmp_path, orc):
    """The NCCL backend on the box's one GPU: process group, stream-ordered
    barrier (all-reduce) and both distributed three-primes entry points.
    World sizes > 1 need one GPU per rank (NCCL rejects two ranks on one
    device); their orchestration is covered by the gloo tests."""
    mp.spawn(_nccl_worker, args=(_free_port(), str(tmp_path)), nprocs=1, join=True)
    want = orc.mul_three_primes(*_inputs(9000, 7001))
    for name in ("nccl_dist", "nccl_p2p"):
        assert np.array_equal(np.load(tmp_path / f"{name}.npy"), want), name
