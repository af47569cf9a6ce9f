"""Benchmark of the modular polynomial-multiplication hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5]
                    [--impl mine|reference]

Default workload = BASELINE.json configs[1] (config 2): a batch of 4096
products of seeded uniform residues mod p = 2013265921, operand lengths
1500 x 2100 -> 3599 coefficients, truncated-transform engine (conv_tft) at
L = 4096.  One step = one batched call over the whole batch.  Under
torchrun each rank multiplies its own 4096-product shard of the seeded stream
(weak scaling, no collective on the data path); value = all ranks' products
/ max-over-ranks device time.

Reported: products/s (metric), Gcoeff/s (output coefficients), the HBM
roofline of the fused kernel (algorithmic bytes 4*(z1+z2+n) per product),
the integer-pipe view (butterflies/s), the end-to-end number through the
public API with host (pinned) buffers, and the CPU baseline = the C oracle
port of the reference path timed on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import os
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

L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def lazy_share(cfg) -> float:
    """Share of the butterflies that run in the lazy-range arithmetic (AR=1,
    p < 2^30 on complete transforms; modarith.cuh): its register pass has a
    higher measured ceiling than the canonical one."""
    if cfg["engine"] == "three_primes":
        return 2.0 / 3.0  # p1, p2 lazy; p3 (31-bit) canonical forward
    n = cfg["z1"] + cfg["z2"] - 1
    L = 1 << (n - 1).bit_length()
    complete = cfg["engine"] == "fft_pad" or -(-n // (L // 16)) == 16
    return 1.0 if (cfg["p"] < (1 << 30) and complete) else 0.0


def _int_roofline(bf: int, pw: int, products_per_s_per_gpu: float, peaks: dict,
                  share_lazy: float = 0.0) -> dict:
    """Integer-pipe roofline: reference butterflies/s per GPU against the
    practical ceiling measured on B200 by scripts/ubench.py (the fused
    kernel's radix-16 register pass in isolation, committed in
    profiles/r01/ubench.json; for the share of butterflies run with lazy
    ranges, the lazy pass's ceiling) and against the nominal IMAD-pipe
    ceiling (64 IMAD/clk/SM, 4 IMAD slots per Shoup butterfly)."""
    achieved = bf * products_per_s_per_gpu
    out = {"bound": "int_pipe", "unit": "butterflies/s", "achieved": achieved,
           "butterflies_per_product": bf, "pointwise_per_product": pw,
           "count": "reference OpCounters butterflies (algorithmic)"}
    try:
        with open(os.path.join(REPO, "profiles", "r01", "ubench.json")) as f:
            ub = json.load(f)
        mhz = float(peaks.get("sm_max_mhz", ub.get("clock_mhz_attr", 1965.0)))
        sms = int(ub.get("sms", 148))
        canon = ub["pass_bf_per_clk_sm_2cta"]
        lazy = max(ub.get("pass_lazy_2p_2cta", canon), ub.get("pass_lazy_2p_alu_2cta", canon))
        # time-weighted: bf/ceiling summed over the two arithmetic modes
        per_clk = 1.0 / (share_lazy / lazy + (1.0 - share_lazy) / canon)
        practical = per_clk * sms * mhz * 1e6
        nominal = 16.0 * sms * mhz * 1e6
        out.update({"peak": practical, "frac": achieved / practical,
                    "peak_kind": ("measured: isolated radix-16 pass, profiles/r01/ubench.json"
                                  f" ({share_lazy:.2f} of the butterflies at the lazy-range pass"
                                  " rate)"),
                    "nominal_peak": nominal, "nominal_frac": achieved / nominal})
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
    per = (time.perf_counter() - t0) / cal
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


def run_reference(args, cfg):
    """--impl reference: the reference path's CPU implementation (the C
    oracle port; the reference itself is pure Python and does not travel to
    the GPU box) with all host threads, same config/metric."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import oracle

    oracle.lib()
    threads = host_threads()
    n = cfg["z1"] + cfg["z2"] - 1
    rates = []
    sample = None
    for i in range(args.warmup + args.steps):
        r, sample, used = cpu_oracle_rate(cfg, threads, target_s=args.ref_step_seconds)
        if i >= args.warmup:
            rates.append(r)
    v = statistics.median(rates)
    line = {
        "impl": "reference", "metric": "modular poly-mults/sec", "value": v,
        "unit": "products/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cfg["batch"] / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded splitmix64)",
        "config": {"workload": cfg["name"], "batch": cfg["batch"], "z1": cfg["z1"],
                   "z2": cfg["z2"], "n": n, "p": cfg["p"], "engine": cfg["engine"]},
        "gcoeff_per_s": v * n / 1e9,
        "cpu_baseline": {"value": v, "unit": "products/s", "cores": used, "kind": "port",
                         "sample": sample + " per step; C restatement of the reference "
                                            "(oracle/modconv_oracle.c)"},
        "e2e": {"value": v, "unit": "products/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_mine(args, cfg):
    import torch

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist

        # BENCH_BACKEND=gloo exercises the multi-rank path on a single GPU
        # (host-side barriers / reductions only; no rank waits on another's
        # kernels).  Production runs use NCCL, one GPU per rank.
        backend = os.environ.get("BENCH_BACKEND", "nccl")
        ngpu = torch.cuda.device_count()
        torch.cuda.set_device(local % ngpu)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    prev_affinity = _bind_local_cpus(torch.cuda.current_device())
    import paper_1609_01010_b200 as mc
    from paper_1609_01010_b200 import _native, _tensors

    lib = _native.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    p, z1, z2, B = cfg["p"], cfg["z1"], cfg["z2"], cfg["batch"]
    n = z1 + z2 - 1
    L = 1 << (n - 1).bit_length()
    engine = cfg["engine"]
    stream = torch.cuda.current_stream()
    sh = _tensors.stream_handle()

    # inputs: this rank's shard of the seeded stream, resident in HBM
    a = torch.empty((B, z1), dtype=torch.int32, device=dev)
    b = torch.empty((B, z2), dtype=torch.int32, device=dev)
    row0 = 0 if engine == "three_primes" else rank * B
    hi = p if engine != "three_primes" else (1 << 30)
    _native.check(lib.mc_gen_u32(cfg["seed"], 0, row0, B, z1, hi, a.data_ptr(), z1, sh))
    _native.check(lib.mc_gen_u32(cfg["seed"], 1, row0, B, z2, hi, b.data_ptr(), z2, sh))
    if engine == "three_primes" and ws > 1:
        # one product, primes spread over the ranks; the residues meet in the
        # CRT: by default each rank's Garner slice reads them from the GPUs
        # that computed them and writes rank 0's limbs over peer memory (the
        # gather fused into the kernel); MC_CRT_NCCL=1 gathers them to rank 0
        # with NCCL send/recv first
        from paper_1609_01010_b200.distributed import (mul_three_primes_distributed,
                                                       mul_three_primes_p2p)

        c = torch.empty((3, n), dtype=torch.int32, device=dev)
        dist_fn = mul_three_primes_distributed if os.environ.get("MC_CRT_NCCL") else mul_three_primes_p2p

        def step():
            dist_fn(a[0], b[0], dst=0)
    elif engine == "three_primes":
        c = torch.empty((3, n), dtype=torch.int32, device=dev)

        def step():
            mc.mul_three_primes_tensor(a[0], b[0], out=c)
    else:
        c = torch.empty((B, n), dtype=torch.int32, device=dev)

        def step():
            mc.conv_batch(a, b, p, engine=engine, out=c)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    # clock sampling starts before the warm-up steps (its start-up pause must
    # not sit between the warm-up and the timed steps: the first kernel after
    # an idle GPU runs at half speed) and runs through the timed region
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    time.sleep(0.3)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    graph = None
    if (B * n <= (1 << 20) and engine != "three_primes") or (engine == "three_primes" and ws == 1):
        # launch-bound workloads (config 1; config 5's ~20 launches and stream-
        # ordered allocations per step): replay the step from a CUDA graph so
        # the timed region measures the device, not the Python launch path
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
        step_eager = step

        def step():
            graph.replay()

        for _ in range(args.warmup):  # the warm-up steps again, now as replays
            flush.zero_()
            step()
        torch.cuda.synchronize()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region: K steps, L2 flushed before each
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
        print("step times (ms):", " ".join(f"{t:.4f}" for t in times), file=sys.stderr)
    total_ms = sum(times)
    t_local = torch.tensor([total_ms], dtype=torch.float64, device=_coll_device(dev))
    if ws > 1:
        torch.distributed.all_reduce(t_local, op=torch.distributed.ReduceOp.MAX)
    t_max = float(t_local.item())
    strong = engine == "three_primes" and ws > 1  # one product shared by all ranks
    products = B * args.steps * (1 if strong else ws)
    value = products / (t_max / 1e3)
    ms_step = t_max / args.steps

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if engine != "three_primes":
        a_h = a.cpu().pin_memory()
        b_h = b.cpu().pin_memory()
        c_h = torch.empty((B, n), dtype=torch.int32).pin_memory()
        for _ in range(max(1, args.warmup)):
            mc.conv_batch(a_h, b_h, p, engine=engine, out=c_h)
        torch.cuda.synchronize()
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        barrier()
        for i in range(args.steps):
            flush.zero_()
            ev2[i][0].record(stream)
            mc.conv_batch(a_h, b_h, p, engine=engine, out=c_h)
            ev2[i][1].record(stream)
        barrier()
        t2 = torch.tensor([sum(s.elapsed_time(e) for s, e in ev2)], dtype=torch.float64,
                          device=_coll_device(dev))
        if ws > 1:
            torch.distributed.all_reduce(t2, op=torch.distributed.ReduceOp.MAX)
        assert torch.equal(c_h.to(dev), c), "e2e output differs from device-resident output"
        e2e = {"value": products / (float(t2.item()) / 1e3), "unit": "products/s",
               "h2d_bytes_per_step": 4 * B * (z1 + z2), "d2h_bytes_per_step": 4 * B * n}
    else:
        a_h = a[0].cpu().pin_memory()
        b_h = b[0].cpu().pin_memory()
        c_h = torch.empty((3, n), dtype=torch.int32).pin_memory()
        mc.mul_three_primes_tensor(a_h, b_h, out=c).cpu()
        torch.cuda.synchronize()
        barrier()
        ev3 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            ev3[i][0].record(stream)
            cc = mc.mul_three_primes_tensor(a_h, b_h, out=c)
            c_h.copy_(cc, non_blocking=True)
            ev3[i][1].record(stream)
        barrier()
        t3 = sum(s.elapsed_time(e) for s, e in ev3)
        e2e = {"value": args.steps / (t3 / 1e3), "unit": "products/s",
               "h2d_bytes_per_step": 4 * (z1 + z2), "d2h_bytes_per_step": 12 * n}

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return

    peak, peak_kind, peaks = _peaks()
    if engine == "three_primes":
        # compulsory I/O plus the four-step pass model per prime
        alg_bytes = 4 * (z1 + z2) + 12 * n + 3 * 4 * 6 * L
        bytes_note = "4*(z1+z2) in + 12*n limbs out + 3 primes x 4*6L four-step passes"
    elif L > 8192:
        alg_bytes = 4 * (z1 + z2 + n + 6 * L) * B
        bytes_note = "four-step pass model 4*(z1+z2+n+6L) per product"
    else:
        alg_bytes = 4 * (z1 + z2 + n) * B
        bytes_note = "compulsory 4*(z1+z2+n) per product (fused single pass)"
    kern_ms = statistics.mean(times)  # one launch of the fused kernel per step (cfg 1-3)
    traffic, ncu_pipes = None, None
    try:  # DRAM bytes and pipe utilisation per launch from the committed ncu capture
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(cfg["name"])
        if tr:
            traffic = tr["dram_bytes_read"] + tr["dram_bytes_write"]
            ncu_pipes = tr.get("ncu_pipes")
    except Exception:
        traffic = None
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    from paper_1609_01010_b200.transform import full_count, itft_count, tft_count

    if engine == "tft":
        bf = tft_count(L, z1, n) + tft_count(L, z2, n) + itft_count(L, n)
        pw = n
    elif engine == "fft_pad":
        bf, pw = 3 * full_count(L), L
    else:
        bf, pw = 3 * 3 * full_count(L), 3 * L
    if prev_affinity:  # the CPU baseline uses every host thread again
        os.sched_setaffinity(0, prev_affinity)
    cpu_rate, sample, cpu_cores = cpu_oracle_rate(cfg, host_threads(), target_s=args.ref_seconds)
    line = {
        "metric": "modular poly-mults/sec", "value": value, "unit": "products/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded splitmix64 uniform residues, generated on device)",
        "config": {"workload": cfg["name"], "batch_per_rank": B, "global_batch": B * ws,
                   "z1": z1, "z2": z2, "n": n, "L": L, "p": p, "engine": engine,
                   "parallelism": f"dp{ws} (independent products)",
                   "l2": "flushed (256 MiB write) before every timed step",
                   "launch": "cuda graph replay" if graph is not None else "eager"},
        "gcoeff_per_s": value * n / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "alg_bytes_per_step": alg_bytes, "bytes_model": bytes_note,
                     "kernel_ms": kern_ms},
        "int_pipe": dict(_int_roofline(bf, pw, value / ws, peaks, lazy_share(cfg)),
                         **({"ncu": ncu_pipes} if ncu_pipes else {})),
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "cpu_baseline": {"value": cpu_rate, "unit": "products/s", "cores": cpu_cores,
                         "kind": "port", "sample": sample},
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--engine", default=None, choices=["tft", "fft_pad"],
                    help="override the config's engine (analysis only)")
    ap.add_argument("--ref-seconds", type=float, default=10.0,
                    help="target CPU seconds of the cpu_baseline sample")
    ap.add_argument("--ref-step-seconds", type=float, default=2.0,
                    help="target CPU seconds per --impl reference step")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.engine:  # analysis override (e.g. fft_pad on config 2's shapes)
        cfg["engine"] = args.engine
        cfg["name"] += f"_engine_{args.engine}"
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_mine(args, cfg)


if __name__ == "__main__":
    main()
