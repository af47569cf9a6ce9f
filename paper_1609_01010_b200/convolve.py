"""Convolution engines over prime fields and the poly_mul dispatcher (GPU).

Call-compatible with the reference's engine functions
(/root/reference/pkg/src/modconv/convolve.py): ConvRequest, ENGINES,
circ_conv_fft (:143-157), lin_conv_fft_pad (:160-169), conv_tft (:230-253)
and poly_mul (:264-296), plus a batched tensor API (conv_batch) that is the
hot path proper: [B, z1] x [B, z2] -> [B, n] in one kernel launch.

Engines run in libmodconv_b200 (mc_conv_fft_pad / mc_conv_tft /
mc_circ_conv / mc_circ_conv_split).  `threads` is accepted and ignored (the
GPU does not use host workers; results are schedule-independent like the
reference's).  The quadratic "definition" engine is a CPU oracle in the
reference; here it is served by the GPU fft_pad kernel where the field has
the roots of unity (bit-identical output, no counters touched, exactly as
lin_conv_def touches none) and by the defining-sum kernel (mc_conv_direct)
beyond the field's 2-adicity, where the reference's definition engine keeps
working too.  The
Eq. 13 "split" engine (nega_conv, circ_conv_split, split_residues,
recombine_residues: convolve.py:172-227) runs on the GPU as two half-length
circular convolutions around fused split/twist and untwist/recombine
kernels.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import torch

from . import _native, _tensors
from .field import FieldMismatchError, FourierPrime, as_field, check_transform_size
from .poly import DensePoly
from .transform import OpCounters, full_count, itft_count, tft_count

ENGINES = ("definition", "fft_pad", "tft", "split", "auto")


@dataclass
class ConvRequest:
    """How to run a convolution (convolve.py:33-47)."""

    field: object
    engine: str = "auto"
    threads: int = 1
    counters: OpCounters | None = None
    planner: object = dc_field(default=None, repr=False)

    def __post_init__(self) -> None:
        if self.engine not in ENGINES:
            raise ValueError(f"unknown engine {self.engine!r}; choose from {ENGINES}")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")


def _next_pow2(n: int) -> int:
    return 1 << (n - 1).bit_length() if n > 1 else 1


def count_engine(engine: str, z1: int, z2: int, counters: OpCounters | None, batch: int = 1):
    """Reference OpCounters for one engine call (per product x batch)."""
    if counters is None:
        return
    n = z1 + z2 - 1
    L = _next_pow2(n)
    if engine == "fft_pad":
        counters.butterflies += 3 * full_count(L) * batch
        counters.pointwise_muls += L * batch
    elif engine == "tft":
        bf = tft_count(L, z1, n) + tft_count(L, z2, n) + itft_count(L, n)
        counters.butterflies += bf * batch
        counters.pointwise_muls += n * batch


# ------------------------------------------------------------------ batched API
def _as_batch(x, name: str) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        raise ValueError(f"{name} must be a torch tensor")
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if x.dim() != 2:
        raise ValueError(f"{name} must be [batch, length]")
    return _tensors.as_words(x)


def _transform_feasible(fp, n: int) -> bool:
    """Whether a power-of-two transform covering n outputs exists in fp
    (log2 L within the 2-adicity) -- else only the definition engine applies."""
    return (_next_pow2(n)).bit_length() - 1 <= fp.two_adicity


def _direct_batch(a_d: torch.Tensor, b_d: torch.Tensor, c_d: torch.Tensor, p: int,
                  circ: bool, stream=None) -> None:
    """Definition engine on device rows (mc_conv_direct), batch-chunked to the
    kernel's grid limit."""
    B = a_d.shape[0]
    z1, z2 = a_d.shape[1], b_d.shape[1]
    lib = _native.lib()
    for r0 in range(0, B, 65535):
        nb = min(65535, B - r0)
        _native.check(lib.mc_conv_direct(
            _tensors.ptr(a_d[r0]), a_d.stride(0), z1, _tensors.ptr(b_d[r0]), b_d.stride(0), z2,
            _tensors.ptr(c_d[r0]), c_d.stride(0), nb, p, 1 if circ else 0,
            _tensors.stream_handle(stream)))


def conv_batch(a: torch.Tensor, b: torch.Tensor, field, engine: str = "tft",
               out: torch.Tensor | None = None, counters: OpCounters | None = None,
               stream=None) -> torch.Tensor:
    """Row-wise linear convolution mod p of a [B, z1] and b [B, z2] -> [B, n].

    Tensors hold canonical residues as int32 (or uint32).  CUDA inputs are
    used in place (rows may be strided: any row stride >= row length);
    CPU inputs are copied to the current device inside the call and the
    result is copied back (the host-buffer path: H2D, kernel, D2H).
    engine: "tft" (truncated transforms, convolve.py:230-253), "fft_pad"
    (zero-padded full transforms, convolve.py:160-169), "definition" (the
    defining sum, convolve.py:71-87; any length, no roots of unity) or
    "auto" (GpuPlanner).
    """
    if stream is not None and stream != torch.cuda.current_stream():
        # every temporary and the output are then allocated on `stream`, and
        # the kernels run there: nothing is freed while `stream` still uses it
        with torch.cuda.stream(stream):
            return conv_batch(a, b, field, engine, out, counters, None)
    if engine not in ("tft", "fft_pad", "definition", "auto"):
        raise ValueError("batched engine must be 'tft', 'fft_pad', 'definition' or 'auto', "
                         f"got {engine!r}")
    fp = as_field(field)
    a = _as_batch(a, "a")
    b = _as_batch(b, "b")
    if a.shape[0] != b.shape[0]:
        raise ValueError(f"batch mismatch: {a.shape[0]} vs {b.shape[0]}")
    B, z1 = a.shape
    z2 = b.shape[1]
    if z1 < 1 or z2 < 1:
        raise ValueError("inputs must be nonempty")
    n = z1 + z2 - 1
    if engine != "definition":
        check_transform_size(fp, (_next_pow2(n)).bit_length() - 1)
    dev = _tensors.require_cuda()
    if engine == "auto":  # GPU-timed choice per size class (planner.GpuPlanner)
        engine = default_planner().resolve_engine(fp, z1, z2)
    host = a.device.type == "cpu"
    if host != (b.device.type == "cpu"):
        raise ValueError("a and b must be on the same device")
    if engine == "definition":
        a_d = a.to(dev) if host else a
        b_d = b.to(dev) if host else b
        if a_d.stride(1) != 1 or b_d.stride(1) != 1:
            a_d, b_d = a_d.contiguous(), b_d.contiguous()
        c_d = torch.empty((B, n), dtype=torch.int32, device=dev)
        _direct_batch(a_d, b_d, c_d, fp.p, False, stream)
        if out is not None:
            _tensors.as_words(out).copy_(c_d)
            return out
        return c_d.cpu() if host else c_d
    if host:
        return _conv_batch_host(a, b, fp, engine, out, counters, stream)
    a_d, b_d = a, b
    if a_d.stride(1) != 1 or b_d.stride(1) != 1:
        a_d, b_d = a_d.contiguous(), b_d.contiguous()
    if out is not None:
        c_d = _tensors.as_words(out)
        if c_d.shape != (B, n) or c_d.stride(1) != 1 or c_d.device != a_d.device:
            raise ValueError(f"out must be a [B, {n}] tensor on {a_d.device} with unit column stride")
    else:
        c_d = torch.empty((B, n), dtype=torch.int32, device=a_d.device)
    fn = _native.lib().mc_conv_tft if engine == "tft" else _native.lib().mc_conv_fft_pad
    _native.check(fn(_tensors.ptr(a_d), a_d.stride(0), z1, _tensors.ptr(b_d), b_d.stride(0), z2,
                     _tensors.ptr(c_d), c_d.stride(0), B, fp.p, _tensors.stream_handle(stream)))
    count_engine(engine, z1, z2, counters, B)
    return c_d


def _conv_batch_host(a, b, fp, engine, out, counters, stream) -> torch.Tensor:
    """Host tensors: chunked H2D / kernel / D2H pipeline on three streams
    (mc_conv_host_async).  Pinned buffers overlap copies in both directions
    with the kernels.  The result is complete when the call returns."""
    B, z1 = a.shape
    z2 = b.shape[1]
    n = z1 + z2 - 1
    a_h = a if a.stride(1) == 1 else a.contiguous()
    b_h = b if b.stride(1) == 1 else b.contiguous()
    if out is not None:
        c_h = _tensors.as_words(out)
        if c_h.shape != (B, n) or c_h.stride(1) != 1 or c_h.device.type != "cpu":
            raise ValueError(f"out must be a CPU [B, {n}] tensor with unit column stride")
    else:
        c_h = torch.empty((B, n), dtype=torch.int32, pin_memory=a_h.is_pinned())
    st = stream if stream is not None else torch.cuda.current_stream()
    _native.check(_native.lib().mc_conv_host_async(
        1 if engine == "tft" else 0, _tensors.ptr(a_h), a_h.stride(0), z1, _tensors.ptr(b_h),
        b_h.stride(0), z2, _tensors.ptr(c_h), c_h.stride(0), B, fp.p, 0, int(st.cuda_stream)))
    st.synchronize()
    count_engine(engine, z1, z2, counters, B)
    return out if out is not None else c_h


_DEFAULT_PLANNER = None


def default_planner():
    """Process-wide GpuPlanner used by conv_batch(engine="auto")."""
    global _DEFAULT_PLANNER
    if _DEFAULT_PLANNER is None:
        from .planner import GpuPlanner

        _DEFAULT_PLANNER = GpuPlanner()
    return _DEFAULT_PLANNER


# ------------------------------------------------------------------ list API
def _run_lists(engine: str, u, v, req: ConvRequest) -> list[int]:
    """One product from Python lists: residues into page-locked staging, the
    zero-copy host call (the kernel reads and writes the staging directly),
    the product read back as ints."""
    fp = as_field(req.field)
    _tensors.require_cuda()
    z1, z2 = len(u), len(v)
    n = z1 + z2 - 1
    oa, ob = 0, (z1 + 3) & ~3  # 16-byte aligned operand rows (bulk copies)
    oc = ob + ((z2 + 3) & ~3)
    st = _tensors.host_stage(oc + n)
    st[oa:oa + z1] = _tensors.words_from_list(u, fp.p)
    st[ob:ob + z2] = _tensors.words_from_list(v, fp.p)
    base = st.ctypes.data
    stream = torch.cuda.current_stream()
    _native.check(_native.lib().mc_conv_host_async(
        1 if engine == "tft" else 0, base + 4 * oa, z1, z1, base + 4 * ob, z2, z2,
        base + 4 * oc, n, 1, fp.p, 0, int(stream.cuda_stream)))
    stream.synchronize()
    return st[oc:oc + n].tolist()


def _direct_lists(u, v, p: int, circ: bool) -> list[int]:
    dev = _tensors.require_cuda()
    a = _tensors.list_to_device(u, p, dev).view(1, -1)
    b = _tensors.list_to_device(v, p, dev).view(1, -1)
    n = len(u) if circ else len(u) + len(v) - 1
    c = torch.empty((1, n), dtype=torch.int32, device=dev)
    _direct_batch(a, b, c, p, circ)
    return _tensors.device_to_list(c[0])


def circ_conv_def(u, v, fp) -> list[int]:
    """Circular convolution straight from its defining sum (convolve.py:54-68),
    on the GPU (mc_conv_direct): any length, any field, no counters."""
    n = len(u)
    if n == 0 or len(v) != n:
        raise ValueError(f"need equal nonempty lengths, got {len(u)} and {len(v)}")
    return _direct_lists(u, v, as_field(fp).p, True)


def lin_conv_def(u, v, fp) -> list[int]:
    """Linear convolution straight from its defining sum (convolve.py:71-87),
    on the GPU (mc_conv_direct): any length, any field, no counters."""
    if len(u) == 0 or len(v) == 0:
        raise ValueError("inputs must be nonempty")
    return _direct_lists(u, v, as_field(fp).p, False)


def circ_conv_fft(u, v, req: ConvRequest) -> list[int]:
    """Circular convolution of two power-of-two length vectors
    (convolve.py:143-157)."""
    n = len(u)
    if n == 0 or len(v) != n:
        raise ValueError(f"need equal nonempty lengths, got {len(u)} and {len(v)}")
    if n & (n - 1):
        raise ValueError(f"length must be a power of two: {n}")
    fp = as_field(req.field)
    check_transform_size(fp, n.bit_length() - 1)
    dev = _tensors.require_cuda()
    a = _tensors.list_to_device(u, fp.p, dev)
    b = _tensors.list_to_device(v, fp.p, dev)
    c = torch.empty_like(a)
    _native.check(_native.lib().mc_circ_conv(_tensors.ptr(a), _tensors.ptr(b), _tensors.ptr(c),
                                             n.bit_length() - 1, 1, fp.p,
                                             _tensors.stream_handle()))
    if req.counters is not None:
        req.counters.butterflies += 3 * full_count(n)
        req.counters.pointwise_muls += n
    return _tensors.device_to_list(c)


def lin_conv_fft_pad(u, v, req: ConvRequest) -> list[int]:
    """Linear convolution by zero-padding to a power of two
    (convolve.py:160-169).  Output not normalized."""
    if len(u) == 0 or len(v) == 0:
        raise ValueError("inputs must be nonempty")
    out = _run_lists("fft_pad", u, v, req)
    count_engine("fft_pad", len(u), len(v), req.counters)
    return out


def conv_tft(g, h, req: ConvRequest) -> list[int]:
    """Linear convolution via truncated transforms (convolve.py:230-253)."""
    if len(g) == 0 or len(h) == 0:
        raise ValueError("inputs must be nonempty")
    out = _run_lists("tft", g, h, req)
    count_engine("tft", len(g), len(h), req.counters)
    return out


# ------------------------------------------------------------------ split engine
def _pow2_len(n: int, what: str = "length") -> int:
    if n == 0 or n & (n - 1):
        raise ValueError(f"{what} must be a power of two: {n}")
    return n.bit_length() - 1


def split_residues(u, p: int) -> tuple[list[int], list[int]]:
    """Residues of u mod (x^n - 1) and mod (x^n + 1), n = len(u) >> 1
    (convolve.py:214-219), on the GPU.  Any length, like the reference: an
    odd length's last coefficient takes no part; power-of-two lengths run the
    fused kernel (mc_split_residues), others device tensor arithmetic."""
    size = len(u)
    n = size >> 1
    dev = _tensors.require_cuda()
    if n == 0:
        return [], []
    x = _tensors.list_to_device(u, p, dev)
    if size & (size - 1):
        lo = x[:n].to(torch.int64)
        hi = x[n:2 * n].to(torch.int64)
        return (_tensors.device_to_list(((lo + hi) % p).to(torch.int32)),
                _tensors.device_to_list(((lo - hi) % p).to(torch.int32)))
    a = torch.empty(n, dtype=torch.int32, device=dev)
    b = torch.empty_like(a)
    _native.check(_native.lib().mc_split_residues(_tensors.ptr(x), _tensors.ptr(a),
                                                  _tensors.ptr(b), n.bit_length() - 1, 1, p,
                                                  _tensors.stream_handle()))
    return _tensors.device_to_list(a), _tensors.device_to_list(b)


def recombine_residues(a, b, p: int) -> list[int]:
    """Inverse of split_residues (convolve.py:222-227), on the GPU: pairs
    (a_j, b_j) up to the shorter length, like the reference's zip."""
    n = min(len(a), len(b))
    dev = _tensors.require_cuda()
    if n == 0:
        return []
    x = _tensors.list_to_device(list(a[:n]), p, dev)
    y = _tensors.list_to_device(list(b[:n]), p, dev)
    if n & (n - 1):
        inv2 = (p + 1) >> 1
        xs, ys = x.to(torch.int64), y.to(torch.int64)
        lo = (xs + ys) % p * inv2 % p
        hi = (xs - ys) % p * inv2 % p
        return _tensors.device_to_list(torch.cat([lo, hi]).to(torch.int32))
    w = torch.empty(2 * n, dtype=torch.int32, device=dev)
    _native.check(_native.lib().mc_recombine_residues(_tensors.ptr(x), _tensors.ptr(y),
                                                      _tensors.ptr(w), n.bit_length() - 1, 1, p,
                                                      _tensors.stream_handle()))
    return _tensors.device_to_list(w)


def nega_conv(u, v, req: ConvRequest) -> list[int]:
    """Negacyclic convolution (product mod x^n + 1) via the psi twist
    (convolve.py:172-190).  Needs 2-adicity >= log2(2n)."""
    n = len(u)
    if n == 0 or len(v) != n:
        raise ValueError(f"need equal nonempty lengths, got {len(u)} and {len(v)}")
    lg = _pow2_len(n)
    fp = as_field(req.field)
    check_transform_size(fp, lg + 1)
    dev = _tensors.require_cuda()
    a = _tensors.list_to_device(u, fp.p, dev)
    b = _tensors.list_to_device(v, fp.p, dev)
    c = torch.empty_like(a)
    _native.check(_native.lib().mc_nega_conv(_tensors.ptr(a), _tensors.ptr(b), _tensors.ptr(c),
                                             lg, 1, fp.p, _tensors.stream_handle()))
    if req.counters is not None:
        req.counters.butterflies += 3 * full_count(n)
        req.counters.pointwise_muls += n
    return _tensors.device_to_list(c)


def circ_conv_split(u, v, req: ConvRequest) -> list[int]:
    """Circular convolution of length 2n via the (x^n - 1)/(x^n + 1) split
    (convolve.py:193-211)."""
    size = len(u)
    if size == 0 or len(v) != size:
        raise ValueError(f"need equal nonempty lengths, got {len(u)} and {len(v)}")
    if size & (size - 1) or size < 2:
        raise ValueError(f"length must be a power of two >= 2: {size}")
    fp = as_field(req.field)
    lg = size.bit_length() - 1
    check_transform_size(fp, lg)
    dev = _tensors.require_cuda()
    a = _tensors.list_to_device(u, fp.p, dev)
    b = _tensors.list_to_device(v, fp.p, dev)
    c = torch.empty_like(a)
    _native.check(_native.lib().mc_circ_conv_split(_tensors.ptr(a), _tensors.ptr(b),
                                                   _tensors.ptr(c), lg, 1, fp.p,
                                                   _tensors.stream_handle()))
    if req.counters is not None:  # circ_conv_fft + nega_conv, both on n points
        n = size // 2
        req.counters.butterflies += 2 * 3 * full_count(n)
        req.counters.pointwise_muls += 2 * n
    return _tensors.device_to_list(c)


def _resolve_engine(a_len: int, b_len: int, req: ConvRequest) -> str:
    if req.engine != "auto":
        return req.engine
    if req.planner is None:
        raise ValueError("engine 'auto' requires a ConvRequest.planner plan session")
    return req.planner.resolve_engine(req.field, a_len, b_len, req.threads)


def poly_mul(a, b, req: ConvRequest) -> DensePoly:
    """Multiply polynomials with the requested engine (convolve.py:264-296).

    Zero inputs short-circuit without touching any transform or counter;
    inputs are normalized first; the result is normalized.  Accepts this
    package's DensePoly or any object with .field.p and .coeffs (e.g. the
    reference's own DensePoly).
    """
    if a.field.p != b.field.p:
        raise FieldMismatchError(f"mixed moduli {a.field.p} and {b.field.p}")
    if a.field.p != req.field.p:
        raise FieldMismatchError(f"request field {req.field.p} does not match operands {a.field.p}")
    fp = as_field(req.field)
    # the result lives on the caller's field and class (convolve.py:277-278,
    # 296): the reference's own DensePoly in, the reference's DensePoly out
    cls = type(a) if hasattr(type(a), "zero") else DensePoly
    if not any(a.coeffs) or not any(b.coeffs):
        return cls.zero(a.field)
    u = _trim(a.coeffs)
    v = _trim(b.coeffs)
    engine = _resolve_engine(len(u), len(v), req)
    if engine == "definition":
        # bit-identical either way: the fused transform kernel where the field
        # has the roots, the defining sum beyond its 2-adicity
        if _transform_feasible(fp, len(u) + len(v) - 1):
            out = _run_lists("fft_pad", u, v, req)
        else:
            out = _direct_lists(u, v, fp.p, False)
    elif engine == "fft_pad":
        out = lin_conv_fft_pad(u, v, req)
    elif engine == "tft":
        out = conv_tft(u, v, req)
    elif engine == "split":
        out_len = len(u) + len(v) - 1
        size = max(2, _next_pow2(out_len))
        up = u + [0] * (size - len(u))
        vp = v + [0] * (size - len(v))
        out = circ_conv_split(up, vp, req)[:out_len]
    else:
        raise ValueError(f"unknown engine {engine!r}")
    if cls is DensePoly:
        # the engines return canonical residues: wrap without re-validating them
        return DensePoly._trusted(a.field if isinstance(a.field, FourierPrime) else fp,
                                  tuple(out)).normalize()
    return cls(a.field, tuple(out)).normalize()


def _trim(coeffs) -> list[int]:
    c = list(coeffs)
    while c and not c[-1]:
        c.pop()
    return c
