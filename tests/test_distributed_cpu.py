"""Multi-rank host logic under gloo on CPU (world size 2 and 3): row
sharding, prime assignment and the config-5 residue gather.  The per-prime
product and the CRT are injected from the oracle (the GPU kernels are
covered by the -m gpu tests)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO

from paper_1609_01010_b200.distributed import primes_of_rank, shard_rows


def test_shard_rows_partition():
    for batch in (0, 1, 7, 4096, 65536):
        for ws in (1, 2, 3, 4, 8):
            spans = [shard_rows(batch, ws, r) for r in range(ws)]
            assert spans[0][0] == 0
            for (r0, n0), (r1, _) in zip(spans, spans[1:]):
                assert r0 + n0 == r1
            assert sum(n for _, n in spans) == batch
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1


def test_primes_of_rank_cover():
    for ws in (1, 2, 3, 4, 8):
        owned = sorted(k for r in range(ws) for k in primes_of_rank(ws, r))
        assert owned == [0, 1, 2]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, out_dir):
    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from oracle import oracle

    from paper_1609_01010_b200.crt import PRIMES
    from paper_1609_01010_b200.distributed import mul_three_primes_distributed

    rng = np.random.default_rng(123)
    a_np = rng.integers(0, 1 << 30, 700, dtype=np.uint64).astype(np.uint32)
    b_np = rng.integers(0, 1 << 30, 500, dtype=np.uint64).astype(np.uint32)
    a = torch.from_numpy(a_np.view(np.int32))
    b = torch.from_numpy(b_np.view(np.int32))
    calls = []

    def prime_product(x, y, k):
        calls.append(k)
        p = PRIMES[k]
        xa = x.numpy().view(np.uint32) % p
        ya = y.numpy().view(np.uint32) % p
        c, _, _ = oracle.conv_batch(xa[None], ya[None], p)
        return torch.from_numpy(c[0].view(np.int32).copy())

    def crt(r1, r2, r3):
        limbs = oracle.crt3(*(r.numpy().view(np.uint32) for r in (r1, r2, r3)))
        return torch.from_numpy(limbs.view(np.int32).copy())

    res = mul_three_primes_distributed(a, b, dst=0, prime_product=prime_product, crt=crt)
    np.save(os.path.join(out_dir, f"calls_{rank}.npy"), np.array(calls))
    if rank == 0:
        np.save(os.path.join(out_dir, "limbs.npy"), res.numpy().view(np.uint32))
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_three_primes_gather_gloo(tmp_path, orc, ws):
    mp.spawn(_worker, args=(ws, _free_port(), str(tmp_path)), nprocs=ws, join=True)
    limbs = np.load(tmp_path / "limbs.npy")
    rng = np.random.default_rng(123)
    a = rng.integers(0, 1 << 30, 700, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 1 << 30, 500, dtype=np.uint64).astype(np.uint32)
    assert np.array_equal(limbs, orc.mul_three_primes(a, b))
    calls = sorted(int(k) for r in range(ws) for k in np.load(tmp_path / f"calls_{r}.npy"))
    assert calls == [0, 1, 2]  # every prime computed exactly once


@pytest.mark.parametrize("ws", [2, 3])
def test_bench_self_launches_ranks(ws):
    """`bench.py --gpus N` outside torchrun re-launches itself with N ranks;
    every config's global batch is partitioned over them (strong scaling):
    the shards tile the batch exactly, config 1 runs as replicas and
    config 5 spreads its primes."""
    import json
    import subprocess

    env = dict(os.environ, BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", str(ws),
                        "--plan-only"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == ws
    cfgs = line["configs"]
    assert list(cfgs)[0] == "cfg2"  # the headline config first
    for name, batch in (("cfg2", 4096), ("cfg3", 65536), ("cfg4", 8)):
        c = cfgs[name]
        assert c["mode"] == "shards"
        assert c["config"]["global_batch"] == batch == c["covered_rows"]
        spans = c["ranges"]
        assert len(spans) == ws and spans[0][0] == 0
        assert all(a[0] + a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert cfgs["cfg1"]["mode"] == "replicas" and cfgs["cfg1"]["global_products"] == ws
    assert cfgs["cfg5"]["mode"] == "primes" and cfgs["cfg5"]["global_products"] == 1


def _barrier_worker(rank, ws, port, out_dir):
    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_1609_01010_b200.distributed import _stream_barrier

    import time

    time.sleep(0.2 * rank)
    _stream_barrier(None, torch.device("cpu"))
    with open(os.path.join(out_dir, f"t{rank}"), "w") as f:
        f.write(repr(time.time()))
    dist.destroy_process_group()


def test_stream_barrier_host_backend(tmp_path):
    """Under a host backend the p2p CRT's barrier meets every rank."""
    mp.spawn(_barrier_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True)
    ts = [float(open(tmp_path / f"t{r}").read()) for r in range(3)]
    assert max(ts) - min(ts) < 0.3
