"""GPU-timed engine selection for engine="auto".

The reference's PlanSession (planner.py:254-452) times CPU decompositions and
picks definition / fft_pad / tft from a cost model (resolve_engine,
planner.py:410-438).  On the GPU both candidate engines are kernels of this
package, so the planner simply times them: for a size class (p, L, NT) it
runs the fused truncated kernel and the padded kernel on a synthetic batch
and keeps the faster one.  Results are identical either way; only time
differs (e.g. at n just past a power of two the truncated engine forms ~half
the spectrum, while at n = 0.88 L the two are within a few percent).

Duck-type compatible with ConvRequest.planner: resolve_engine(field, a_len,
b_len, threads) -> "fft_pad" | "tft" | "definition" (the last where the
field has no transform of the needed size, or for a single coefficient).
"""

from __future__ import annotations

import json
import os
import threading

import torch

from . import _native
from .field import as_field


class GpuPlanner:
    def __init__(self, batch: int = 256, reps: int = 3, store_path: str | None = None):
        self.batch = batch
        self.reps = reps
        self.store_path = store_path
        self._plans: dict[str, str] = {}
        self._timings: dict[str, dict[str, float]] = {}
        self._lock = threading.Lock()
        self.search_count = 0
        if store_path and os.path.exists(store_path):
            with open(store_path) as f:
                self._plans.update(json.load(f).get("plans", {}))

    @staticmethod
    def size_class(p: int, a_len: int, b_len: int) -> str:
        n = a_len + b_len - 1
        L = 1 << (n - 1).bit_length() if n > 1 else 1
        if L >= 16:
            g = L // 16
            nt = -(-n // g)
        else:
            nt = n
        return f"{p}:{L}:{nt}"

    def _time(self, engine: str, p: int, a_len: int, b_len: int) -> float:
        from .convolve import conv_batch

        dev = torch.device("cuda", torch.cuda.current_device())
        B = max(1, self.batch if (a_len + b_len) <= 16384 else 4)
        a = torch.empty((B, a_len), dtype=torch.int32, device=dev)
        b = torch.empty((B, b_len), dtype=torch.int32, device=dev)
        lib = _native.lib()
        sh = torch.cuda.current_stream().cuda_stream
        _native.check(lib.mc_gen_u32(91, 0, 0, B, a_len, p, a.data_ptr(), a_len, sh))
        _native.check(lib.mc_gen_u32(91, 1, 0, B, b_len, p, b.data_ptr(), b_len, sh))
        out = torch.empty((B, a_len + b_len - 1), dtype=torch.int32, device=dev)
        conv_batch(a, b, p, engine=engine, out=out)  # warm-up (tables, attributes)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = float("inf")
        for _ in range(self.reps):
            s.record()
            conv_batch(a, b, p, engine=engine, out=out)
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e))
        return best

    def resolve_engine(self, field, a_len: int, b_len: int, threads: int = 1) -> str:
        fp = as_field(field)
        p = fp.p
        n = a_len + b_len - 1
        if n == 1 or (n - 1).bit_length() > fp.two_adicity:
            # no transform of that size in this field (or nothing to transform):
            # the defining sum, as the reference's resolve_engine (planner.py:420-422)
            return "definition"
        key = self.size_class(p, a_len, b_len)
        with self._lock:
            hit = self._plans.get(key)
        if hit is not None:
            return hit
        t = {eng: self._time(eng, p, a_len, b_len) for eng in ("tft", "fft_pad")}
        choice = "tft" if t["tft"] <= t["fft_pad"] else "fft_pad"
        with self._lock:
            self._plans[key] = choice
            self._timings[key] = t
            self.search_count += 1
            if self.store_path:
                tmp = self.store_path + ".tmp"
                with open(tmp, "w") as f:
                    json.dump({"format": "modconv-b200-plan v1", "plans": self._plans,
                               "timings_ms": self._timings}, f, indent=1)
                os.replace(tmp, self.store_path)  # atomic, like store_save
        return choice

    def timings(self) -> dict:
        return dict(self._timings)
