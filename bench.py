"""Benchmark of the modular polynomial-multiplication hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5]
                    [--configs 1,2,3,4,5] [--impl mine|reference] [--plan-only]

Headline (`value`) = BASELINE.json configs[1] (config 2): 4096 products of
seeded uniform residues mod p = 2013265921, operand lengths 1500 x 2100 ->
3599 coefficients, truncated-transform engine (conv_tft) at L = 4096.  One
step = one batched call over the whole batch.  The same run times every
other BASELINE config the same way (device-resident inputs, L2 flushed
before every timed step, CUDA events on the launching stream, pinned-host
e2e through the public API, CPU baseline) and reports them under
`all_configs`.

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run (N ranks, 127.0.0.1), one process per GPU over NCCL.
Each config's global batch is partitioned over the ranks (strong scaling,
distributed.shard_rows): config 2 4096/N, config 3 65536/N, config 4 8/N;
config 1 (one product) runs as replicas; config 5 spreads the three primes
over the ranks and fuses the residue gather into the CRT kernel over peer
memory.  Time = max over ranks of the CUDA-event time between barriers;
value = the config's global products / that time.

Reported per config: products/s, Gcoeff/s (output coefficients), the HBM
roofline (compulsory bytes 4*(z1+z2+n) per product for the fused kernel,
the four-step pass model 4*(z1+z2+n+6L) for configs 4-5), the integer-pipe
view against the nominal 16 butterflies/clk/SM and the measured practical
ceiling, the end-to-end rate through the public API with pinned host
buffers, and the CPU baseline = the C oracle port of the reference path on
this host's cores.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

P1, P2, P3 = 469762049, 998244353, 2013265921

CONFIGS = {
    1: dict(name="cfg1_single_1024x1024_p469762049_fft_pad", p=P1, z1=1024, z2=1024, batch=1,
            engine="fft_pad", seed=1),
    2: dict(name="cfg2_tft_batch4096_1500x2100_p2013265921", p=P3, z1=1500, z2=2100,
            batch=4096, engine="tft", seed=2),
    3: dict(name="cfg3_fft_pad_batch65536_4096x4096_p998244353", p=P2, z1=4096, z2=4096,
            batch=65536, engine="fft_pad", seed=3),
    4: dict(name="cfg4_fft_pad_batch8_2^22x2^22_p2013265921", p=P3, z1=1 << 22, z2=1 << 22,
            batch=8, engine="fft_pad", seed=4),
    5: dict(name="cfg5_three_primes_2^20x2^20_crt", p=0, z1=1 << 20, z2=1 << 20, batch=1,
            engine="three_primes", seed=5),
}
HEADLINE = 2
METRIC = "modular poly-mults/sec"

L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def tft_schedule(cfg) -> str:
    """How the library runs a config's product (capi.cu conv_dispatch /
    split_tft_on / tft_full_from, restated): the truncated engine's
    schedule depends on how far n lies past L/2."""
    if cfg["engine"] == "three_primes":
        return "three primes: four-step per prime on forked streams + fused inverse/CRT pass"
    n = cfg["z1"] + cfg["z2"] - 1
    K = (n - 1).bit_length()
    L, G = 1 << K, 1 << max(0, K - 4)
    if cfg["engine"] != "tft" or K <= 3:
        return "complete transforms (fused)" if K <= 13 else "complete transforms (four-step)"
    m = n - L // 2
    lim = L // (16 if K <= 10 else 8)
    big = K >= 10 or cfg["batch"] * L >= (1 << 20)
    if K in (13, 14) and L // 8 < m <= L // 4:
        return f"split truncated product: L/2-point head + twisted L/4-point piece (m = {m})"
    if 5 <= K <= 27 and 1 <= m <= lim and 2 * m - 1 <= 8192 and big:
        return f"split truncated product: L/2-point head + low-product tail (m = {m})"
    nt = -(-n // G)
    if K <= 13:
        if nt >= (13 if K == 13 else 11):
            return (f"complete transform: {nt} of 16 blocks rounded up to 16 (the truncated "
                    "kernel is slower there, DESIGN.md section 3)")
        return f"relaxed truncation: {nt} of 16 blocks (fused)"
    return f"relaxed truncation: {nt} of 16 column blocks (four-step)"


def lazy_share(cfg) -> float:
    """Share of the butterflies that run in the lazy-range arithmetic (AR=1,
    p < 2^30; modarith.cuh): its register pass has a higher measured ceiling
    than the canonical one.  The fused kernels use it for truncated and
    complete transforms, the four-step passes for complete ones."""
    if cfg["engine"] == "three_primes":
        return 2.0 / 3.0  # p1, p2 lazy; p3 (31-bit) canonical forward
    n = cfg["z1"] + cfg["z2"] - 1
    L = 1 << (n - 1).bit_length()
    complete = (cfg["engine"] == "fft_pad" or L <= 8192
                or "truncation" not in tft_schedule(cfg))
    return 1.0 if (cfg["p"] < (1 << 30) and complete) else 0.0


def _int_roofline(bf: int, pw: int, products_per_s_per_gpu: float, peaks: dict,
                  share_lazy: float = 0.0) -> dict:
    """Integer-pipe roofline: reference butterflies/s per GPU against the
    nominal ceiling first (`peak`, `frac`: 16 butterflies/clk/SM -- a
    canonical butterfly needs 4 ALU and 4 FMA-heavy issue slots, both pipes
    at 0.5 warp-instructions/clk/SMSP), then against the practical ceiling
    measured on B200 by scripts/ubench.py (`practical_*`: the fused
    kernel's radix-16 register pass in isolation, profiles/r02/ubench_r02.json;
    for the share of butterflies run with lazy ranges, the lazy pass's
    ceiling) -- a self-measured reference, so it is reported second."""
    achieved = bf * products_per_s_per_gpu
    out = {"bound": "int_pipe", "unit": "butterflies/s", "achieved": achieved,
           "butterflies_per_product": bf, "pointwise_per_product": pw,
           "count": "reference OpCounters butterflies (algorithmic)"}
    try:
        with open(os.path.join(REPO, "profiles", "r02", "ubench_r02.json")) as f:
            ub = json.load(f)
        mhz = float(peaks.get("sm_max_mhz", ub.get("clock_mhz_attr", 1965.0)))
        sms = int(ub.get("sms", 148))
        canon = ub["pass_bf_per_clk_sm_2cta"]
        lazy = max(ub.get("pass_lazy_2p_2cta", canon), ub.get("pass_lazy_2p_alu_2cta", canon))
        # time-weighted: bf/ceiling summed over the two arithmetic modes
        per_clk = 1.0 / (share_lazy / lazy + (1.0 - share_lazy) / canon)
        practical = per_clk * sms * mhz * 1e6
        nominal = 16.0 * sms * mhz * 1e6
        out.update({"peak": nominal, "frac": achieved / nominal,
                    "peak_kind": "nominal: 16 butterflies/clk/SM x 148 SMs x max SM clock",
                    "practical_peak": practical, "practical_frac": achieved / practical,
                    "practical_kind": ("measured: isolated radix-16 pass, "
                                       "profiles/r02/ubench_r02.json"
                                       f" ({share_lazy:.2f} of the butterflies at the lazy-range"
                                       " pass rate)")})
    except Exception:
        pass
    return out


def _bind_local_cpus(dev_index: int):
    """Pin this rank to the CPU cores local to its GPU (NVML affinity), so the
    page-locked buffers of the e2e leg are allocated on the GPU's NUMA node
    and zero-copy / copy-engine traffic does not cross the socket
    interconnect.  Returns the previous affinity (restored for the CPU
    baseline), or None when NVML or the mapping is unavailable."""
    try:
        import pynvml
        import torch

        prop = torch.cuda.get_device_properties(dev_index)
        pynvml.nvmlInit()
        bus = f"{prop.pci_domain_id:08x}:{prop.pci_bus_id:02x}:{prop.pci_device_id:02x}.0"
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        ncpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        old = set(os.sched_getaffinity(0))
        cpus &= old
        if cpus and cpus != old:
            os.sched_setaffinity(0, cpus)
            return old
    except Exception:
        pass
    return None


def _coll_device(dev):
    """Device for collective tensors: the GPU under NCCL, the host under gloo."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_backend() != "nccl":
        return "cpu"
    return dev


def _peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", d
    except Exception:
        return 6650.0, "fallback", {}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sms.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "samples": len(sms), "reasons": sorted(reasons)}


def cpu_oracle_rate(cfg, threads: int, target_s: float = 10.0, max_products=None):
    """Time the C oracle port of the reference path (products/s) on a
    bounded sample of the workload.  Returns (products/s, sample description,
    threads actually used)."""
    from oracle import oracle

    p, z1, z2 = cfg["p"], cfg["z1"], cfg["z2"]
    if cfg["engine"] == "three_primes":
        a = oracle.gen_u32(cfg["seed"], 0, 0, 1, z1, 1 << 30)[0]
        b = oracle.gen_u32(cfg["seed"], 1, 0, 1, z2, 1 << 30)[0]
        used = min(3, threads)  # one thread per prime, serial Garner
        t0 = time.perf_counter()
        oracle.mul_three_primes(a, b, threads=used)
        dt = time.perf_counter() - t0
        return 1.0 / dt, (f"1 three-primes product (3 x fft_pad 2^21 + Garner), "
                          f"{used} threads (one per prime)"), used
    engine = oracle.ENGINE_TFT if cfg["engine"] == "tft" else oracle.ENGINE_FFT_PAD
    B = cfg["batch"]
    # calibrate on a small slice
    cal = max(1, min(B, threads))
    a = oracle.gen_u32(cfg["seed"], 0, 0, cal, z1, p)
    b = oracle.gen_u32(cfg["seed"], 1, 0, cal, z2, p)
    t0 = time.perf_counter()
    oracle.conv_batch(a, b, p, engine, threads=threads)
    dt = time.perf_counter() - t0
    per = dt / cal
    if dt >= 0.5 * target_s or cal == B:  # the calibration slice is the sample
        return cal / dt, f"{cal} of {B} products (rows 0..{cal - 1}), {threads} threads", threads
    nsamp = int(min(B, max(cal, target_s / max(per, 1e-9))))
    if max_products:
        nsamp = min(nsamp, max_products)
    a = oracle.gen_u32(cfg["seed"], 0, 0, nsamp, z1, p)
    b = oracle.gen_u32(cfg["seed"], 1, 0, nsamp, z2, p)
    t0 = time.perf_counter()
    oracle.conv_batch(a, b, p, engine, threads=threads)
    dt = time.perf_counter() - t0
    return nsamp / dt, f"{nsamp} of {B} products (rows 0..{nsamp - 1}), {threads} threads", threads


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1




# ----------------------------------------------------------------- workload
def config_dict(cfg) -> dict:
    """The workload, identical in both arms (and at every N)."""
    n = cfg["z1"] + cfg["z2"] - 1
    d = {"workload": cfg["name"], "global_batch": cfg["batch"], "z1": cfg["z1"],
         "z2": cfg["z2"], "n": n, "L": 1 << (n - 1).bit_length(), "engine": cfg["engine"]}
    if cfg["engine"] == "three_primes":
        d["p"] = [P1, P2, P3]
        d["input_bound"] = 1 << 30
    else:
        d["p"] = cfg["p"]
    return d


def partition(cfg, ws: int, rank: int) -> tuple[int, int, str]:
    """(row0, rows, mode) of this rank's share of the config's global batch.

    shards   -- contiguous rows of the batch (distributed.shard_rows): strong
                scaling, no collective on the data path;
    replicas -- a single product (config 1): every rank multiplies its own
                copy (replicas only; value counts every rank's product);
    primes   -- config 5: one product, its three primes spread over ranks."""
    from paper_1609_01010_b200.distributed import shard_rows

    if cfg["engine"] == "three_primes":
        return 0, 1, "primes"
    if cfg["batch"] == 1:
        return 0, 1, "replicas"
    row0, rows = shard_rows(cfg["batch"], ws, rank)
    return row0, rows, "shards"


def global_products(cfg, ws: int, mode: str) -> int:
    return ws if mode == "replicas" else cfg["batch"]


def bytes_model(cfg) -> tuple[int, str]:
    """Algorithmic bytes per step over the whole global batch."""
    z1, z2, B = cfg["z1"], cfg["z2"], cfg["batch"]
    n = z1 + z2 - 1
    L = 1 << (n - 1).bit_length()
    if cfg["engine"] == "three_primes":
        return (4 * (z1 + z2) + 12 * n + 3 * 4 * 6 * L,
                "4*(z1+z2) in + 12*n limbs out + 3 primes x 4*6L four-step passes")
    if L > 8192:
        return 4 * (z1 + z2 + n + 6 * L) * B, "four-step pass model 4*(z1+z2+n+6L) per product"
    return 4 * (z1 + z2 + n) * B, "compulsory 4*(z1+z2+n) per product (fused single pass)"


def butterflies(cfg) -> tuple[int, int]:
    """Reference OpCounters per product (butterflies, pointwise products)."""
    from paper_1609_01010_b200.transform import full_count, itft_count, tft_count

    n = cfg["z1"] + cfg["z2"] - 1
    L = 1 << (n - 1).bit_length()
    if cfg["engine"] == "tft":
        return (tft_count(L, cfg["z1"], n) + tft_count(L, cfg["z2"], n) + itft_count(L, n), n)
    if cfg["engine"] == "fft_pad":
        return 3 * full_count(L), L
    return 3 * 3 * full_count(L), 3 * L


# ----------------------------------------------------------------- launcher
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args) -> int:
    """--gpus N outside torchrun: run this script under torch.distributed.run
    with N ranks on this node (one process per GPU), rendezvous on
    127.0.0.1.  Returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def init_dist(ws: int, local: int, gpu: bool):
    if ws <= 1:
        return
    import torch
    import torch.distributed as dist

    # BENCH_BACKEND=gloo: host-side collectives only (CPU tests, --plan-only)
    backend = os.environ.get("BENCH_BACKEND", "nccl" if gpu else "gloo")
    if backend == "nccl":
        torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    else:
        if gpu:
            torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group("gloo")


def _allreduce(vals: list, op: str, dev) -> list:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return vals
    t = torch.tensor(vals, dtype=torch.float64, device=_coll_device(dev))
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.tolist()


def plan_only(args, cfg_ids) -> None:
    """--plan-only: the multi-rank plumbing without kernels (runs on CPU):
    rank count, every rank's partition of each config, and the sum of the
    shards, which must equal each config's global batch."""
    ws, rank, local = _dist()
    init_dist(ws, local, gpu=False)
    out = {}
    for c in cfg_ids:
        cfg = CONFIGS[c]
        row0, rows, mode = partition(cfg, ws, rank)
        ranges = [[row0, rows]]
        if ws > 1:
            import torch.distributed as dist

            allr = [None] * ws
            dist.all_gather_object(allr, [row0, rows], group=None)
            ranges = allr
        covered = sum(r[1] for r in ranges) if mode == "shards" else cfg["batch"]
        out[f"cfg{c}"] = {"mode": mode, "ranges": ranges, "covered_rows": covered,
                          "global_products": global_products(cfg, ws, mode),
                          "config": config_dict(cfg)}
    if rank == 0:
        print(json.dumps({"plan_only": True, "n_gpus": ws, "configs": out}), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


# ----------------------------------------------------------------- GPU arm
def measure(cfg, args, ws: int, rank: int) -> dict:
    """Device-resident timed steps, then the pinned-host e2e steps, of one
    config on this rank's partition.  Returns the config's record (rank 0's
    copy carries the max-over-ranks times)."""
    import torch

    import paper_1609_01010_b200 as mc
    from paper_1609_01010_b200 import _native, _tensors

    lib = _native.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    p, z1, z2 = cfg["p"], cfg["z1"], cfg["z2"]
    n = z1 + z2 - 1
    engine = cfg["engine"]
    row0, rows, mode = partition(cfg, ws, rank)
    stream = torch.cuda.current_stream()
    sh = _tensors.stream_handle()
    hi = p if engine != "three_primes" else (1 << 30)

    a = torch.empty((max(rows, 1), z1), dtype=torch.int32, device=dev)
    b = torch.empty((max(rows, 1), z2), dtype=torch.int32, device=dev)
    if rows:
        _native.check(lib.mc_gen_u32(cfg["seed"], 0, row0, rows, z1, hi, a.data_ptr(), z1, sh))
        _native.check(lib.mc_gen_u32(cfg["seed"], 1, row0, rows, z2, hi, b.data_ptr(), z2, sh))
    a, b = a[:rows], b[:rows]
    if engine == "three_primes":
        c = torch.empty((3, n), dtype=torch.int32, device=dev)
        if ws > 1:
            from paper_1609_01010_b200.distributed import mul_three_primes_p2p

            def step(x=a[0], y=b[0]):
                r = mul_three_primes_p2p(x, y, dst=0)
                if r is not None:
                    c.copy_(r)
        else:
            def step(x=a[0], y=b[0]):
                mc.mul_three_primes_tensor(x, y, out=c)
    else:
        c = torch.empty((rows, n), dtype=torch.int32, device=dev)

        def step(x=a, y=b):
            if rows:
                mc.conv_batch(x, y, p, engine=engine, out=c)

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    # clock sampling starts before the warm-up (its start-up pause must not
    # sit between the warm-up and the timed steps) and runs through the
    # timed region
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    time.sleep(0.3)
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    graph = None
    launches_per_step = None
    if rows and ((rows * n <= (1 << 20) and engine != "three_primes")
                 or (engine == "three_primes" and ws == 1)):
        # launch-bound workloads (config 1; config 5's launches and stream-
        # ordered allocations): replay the step from a CUDA graph so the timed
        # region measures the device, not the Python launch path
        l0 = _native.launch_count()
        step()
        launches_per_step = _native.launch_count() - l0
        torch.cuda.synchronize()
        eager_out = c.clone()
        c.zero_()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(c, eager_out), "graph replay differs from the eager step"
        del eager_out

        def step():
            graph.replay()

        for _ in range(args.warmup):  # the warm-up again, now as replays
            flush.zero_()
            step()
        torch.cuda.synchronize()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = _native.launch_count()
    barrier()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    barrier()
    launches = _native.launch_count() - launches0
    if graph is not None:  # replays do not pass through the host launch counter
        launches = launches_per_step * args.steps
    clk = clocks.stop()
    times = [s.elapsed_time(e) for s, e in ev]  # ms
    if os.environ.get("BENCH_STEP_TIMES"):
        print(cfg["name"], "step times (ms):", " ".join(f"{t:.4f}" for t in times),
              file=sys.stderr)
    t_max = _allreduce([sum(times)], "max", dev)[0]
    launches_all, rows_all = _allreduce([float(launches), float(rows)], "sum", dev)
    products = global_products(cfg, ws, mode)
    value = products * args.steps / (t_max / 1e3)

    # ---- end to end through the public API with pinned host buffers
    if engine != "three_primes":
        a_h = a.cpu().pin_memory()
        b_h = b.cpu().pin_memory()
        c_h = torch.empty((rows, n), dtype=torch.int32).pin_memory()

        def e2e_step():
            if rows:
                mc.conv_batch(a_h, b_h, p, engine=engine, out=c_h)
        h2d, d2h = 4 * cfg["batch"] * (z1 + z2), 4 * cfg["batch"] * n
        if mode == "replicas":
            h2d, d2h = h2d * ws, d2h * ws
    else:
        a_h = a[0].cpu().pin_memory()
        b_h = b[0].cpu().pin_memory()
        c_h = torch.empty((3, n), dtype=torch.int32).pin_memory()
        if ws > 1:
            from paper_1609_01010_b200.distributed import mul_three_primes_p2p

            def e2e_step():
                x = a_h.to(dev, non_blocking=True)
                y = b_h.to(dev, non_blocking=True)
                r = mul_three_primes_p2p(x, y, dst=0)
                if r is not None:
                    c_h.copy_(r, non_blocking=True)
        else:
            def e2e_step():
                c_h.copy_(mc.mul_three_primes_tensor(a_h, b_h, out=c), non_blocking=True)
        h2d, d2h = 4 * (z1 + z2) * ws, 12 * n
    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    barrier()
    for i in range(args.steps):
        flush.zero_()
        ev2[i][0].record(stream)
        e2e_step()
        ev2[i][1].record(stream)
    barrier()
    t2 = _allreduce([sum(s.elapsed_time(e) for s, e in ev2)], "max", dev)[0]
    if rows and (engine != "three_primes" or rank == 0):
        assert torch.equal(c_h.to(dev), c), "e2e output differs from the device-resident output"
    e2e = {"value": products * args.steps / (t2 / 1e3), "unit": "products/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "path": "conv_batch on page-locked host tensors (mc_conv_host_async)"
           if engine != "three_primes" else
           "pinned host inputs -> mul_three_primes -> pinned host limbs"}
    del a, b, c, flush, a_h, b_h, c_h
    graph = None
    torch.cuda.empty_cache()

    alg, note = bytes_model(cfg)
    kern_ms = t_max / args.steps  # max-over-ranks device time per step
    peak, peak_kind, peaks = _peaks()
    # per GPU: the bytes this rank's share moved / its step time (ranks equal
    # to within one product)
    alg_gpu = alg if mode == "replicas" else alg / ws
    achieved = alg_gpu / (kern_ms / 1e3) / 1e9
    bf, pw = butterflies(cfg)
    rec = {
        "config": config_dict(cfg),
        "partition": {"mode": mode, "ranks": ws, "rows_this_rank": rows,
                      "rows_all_ranks": int(rows_all)},
        "ms_per_step": kern_ms, "value": value, "unit": "products/s",
        "gcoeff_per_s": value * n / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind,
                     "alg_bytes_per_step": alg, "bytes_model": note, "kernel_ms": kern_ms,
                     "per": "GPU"},
        "int_pipe": _int_roofline(bf, pw, value / ws, peaks, lazy_share(cfg)),
        "e2e": e2e,
        "gpu_launches": int(launches_all),
        "launch": "cuda graph replay" if launches_per_step is not None else "eager",
        "schedule": tft_schedule(cfg),
        "clocks": clk,
    }
    try:  # DRAM bytes and pipe utilisation per launch from a committed ncu capture
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(cfg["name"])
        if tr:
            rec["roofline"]["traffic"] = tr["dram_bytes_read"] + tr["dram_bytes_write"]
            rec["roofline"]["traffic_source"] = tr.get("source")
            if tr.get("ncu_pipes"):
                rec["int_pipe"]["ncu"] = tr["ncu_pipes"]
    except Exception:
        pass
    rec["roofline"].setdefault("traffic", None)
    return rec


def run_mine(args, cfg_ids) -> None:
    import torch

    ws, rank, local = _dist()
    init_dist(ws, local, gpu=True)
    if ws <= 1:
        torch.cuda.set_device(0)
    prev_affinity = _bind_local_cpus(torch.cuda.current_device())
    recs = {c: measure(CONFIGS[c], args, ws, rank) for c in cfg_ids}
    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    if prev_affinity:  # the CPU baselines use every host thread again
        os.sched_setaffinity(0, prev_affinity)
    for c in cfg_ids:
        tgt = args.ref_seconds if c == args.config else args.ref_seconds_other
        rate, sample, cores = cpu_oracle_rate(CONFIGS[c], host_threads(), target_s=tgt)
        recs[c]["cpu_baseline"] = {"value": rate, "unit": "products/s", "cores": cores,
                                   "kind": "port", "sample": sample}
    head = recs[args.config]
    strong = head["partition"]["mode"] != "replicas"
    line = {
        "metric": METRIC, "value": head["value"], "unit": "products/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded splitmix64 uniform residues, generated on device)",
        "config": head["config"],
        "run": {"partition": head["partition"],
                "parallelism": f"{ws} rank(s), one GPU each; "
                               + {"shards": "global batch partitioned (no collective)",
                                  "replicas": "replicas",
                                  "primes": "primes over ranks, CRT gather over peer memory"}[
                                   head["partition"]["mode"]],
                "l2": "flushed (256 MiB write) before every timed step",
                "launch": head["launch"], "timing": "CUDA events, max over ranks"},
        "gcoeff_per_s": head["gcoeff_per_s"],
        "roofline": head["roofline"], "int_pipe": head["int_pipe"], "e2e": head["e2e"],
        "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
        "cpu_baseline": head["cpu_baseline"],
        "all_configs": {f"cfg{c}": recs[c] for c in cfg_ids},
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


# ----------------------------------------------------------------- reference arm
def run_reference(args, cfg_ids) -> None:
    """--impl reference: the reference path's CPU implementation (the C
    oracle port; the reference itself is pure Python and does not travel to
    the GPU box) with all host threads, on the same configs, metric and
    config dicts as the GPU arm.  Under torchrun only rank 0 runs."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import oracle

    oracle.lib()
    threads = host_threads()
    cfg = CONFIGS[args.config]
    rates, sample, used = [], None, threads
    for i in range(args.warmup + args.steps):
        r, sample, used = cpu_oracle_rate(cfg, threads, target_s=args.ref_step_seconds)
        if i >= args.warmup:
            rates.append(r)
    v = statistics.median(rates)
    others = {}
    for c in cfg_ids:
        if c == args.config:
            continue
        r, s, u = cpu_oracle_rate(CONFIGS[c], threads, target_s=args.ref_seconds_other)
        others[f"cfg{c}"] = {"config": config_dict(CONFIGS[c]), "value": r, "unit": "products/s",
                             "cpu_baseline": {"value": r, "unit": "products/s", "cores": u,
                                              "kind": "port", "sample": s}}
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "products/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cfg["batch"] / v, "higher_is_better": True,
        "scaling": "strong" if cfg["batch"] > 1 or cfg["engine"] == "three_primes" else "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded splitmix64)",
        "config": config_dict(cfg),
        "gcoeff_per_s": v * (cfg["z1"] + cfg["z2"] - 1) / 1e9,
        "cpu_baseline": {"value": v, "unit": "products/s", "cores": used, "kind": "port",
                         "sample": sample + " per step; C restatement of the reference "
                                            "(oracle/modconv_oracle.c)"},
        "e2e": {"value": v, "unit": "products/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "all_configs": dict({f"cfg{args.config}": {"config": config_dict(cfg), "value": v,
                                                    "unit": "products/s"}}, **others),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=HEADLINE, choices=sorted(CONFIGS),
                    help="the config of the top-level line")
    ap.add_argument("--configs", default="1,2,3,4,5",
                    help="configs measured in the run (all_configs); 'head' = --config only")
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--engine", default=None, choices=["tft", "fft_pad"],
                    help="override the headline config's engine (analysis only)")
    ap.add_argument("--plan-only", action="store_true",
                    help="multi-rank partition plumbing only, no kernels (CPU)")
    ap.add_argument("--ref-seconds", type=float, default=10.0,
                    help="target CPU seconds of the headline cpu_baseline sample")
    ap.add_argument("--ref-seconds-other", type=float, default=4.0,
                    help="target CPU seconds of the other configs' cpu_baseline samples")
    ap.add_argument("--ref-step-seconds", type=float, default=2.0,
                    help="target CPU seconds per --impl reference step")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    ids = [args.config] if args.configs == "head" else \
        [int(x) for x in args.configs.split(",") if x.strip()]
    if args.config not in ids:
        ids.insert(0, args.config)
    ids = [args.config] + [c for c in ids if c != args.config]  # headline first
    if args.engine:  # analysis override (e.g. fft_pad on config 2's shapes)
        CONFIGS[args.config] = dict(CONFIGS[args.config], engine=args.engine,
                                    name=CONFIGS[args.config]["name"] + f"_engine_{args.engine}")
    if args.plan_only:
        plan_only(args, ids)
    elif args.impl == "reference":
        run_reference(args, ids)
    else:
        run_mine(args, ids)


if __name__ == "__main__":
    main()
