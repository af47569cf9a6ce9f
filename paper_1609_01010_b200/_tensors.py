"""Tensor plumbing between Python containers, torch and the C ABI.

Residues travel as torch.int32 (bit pattern of the uint32 residue; every
residue < 2^31) in contiguous CUDA tensors.  torch is used for device memory
and streams only; all arithmetic happens in the native kernels.
"""

from __future__ import annotations

import array
import threading

import numpy as np
import torch

_U32 = getattr(torch, "uint32", None)


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the modular-convolution path runs on CUDA only (no CPU fallback); "
                           "no CUDA device is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def as_words(t: torch.Tensor) -> torch.Tensor:
    """View a uint32/int32 tensor as int32 words (no copy)."""
    if t.dtype == torch.int32:
        return t
    if _U32 is not None and t.dtype == _U32:
        return t.view(torch.int32)
    raise ValueError(f"expected an int32/uint32 tensor, got {t.dtype}")


def words_from_list(values, p: int) -> np.ndarray:
    """Python ints -> uint32 residues (numpy).  array('I') converts in C when
    every value is a 32-bit word (then one vectorised reduction); other ints
    (negative, >= 2^32) take the element-wise % p path.  Reducing first is
    value-preserving: the reference's arithmetic is mod p throughout."""
    try:
        x = np.frombuffer(array.array("I", values), dtype=np.uint32)
    except (OverflowError, TypeError):
        return np.fromiter((int(v) % p for v in values), dtype=np.uint32, count=len(values))
    if x.size and int(x.max()) >= p:
        x = x % np.uint32(p)
    return x


_STAGE = threading.local()


def host_stage(words: int) -> np.ndarray:
    """Per-thread page-locked staging (uint32 numpy view of a pinned torch
    buffer, grown on demand): the list API hands it to the zero-copy host
    path, so a single product costs one kernel launch and no copies."""
    buf = getattr(_STAGE, "buf", None)
    if buf is None or buf.numel() < words:
        buf = torch.empty(max(words, 1 << 16), dtype=torch.int32).pin_memory()
        _STAGE.buf = buf
        _STAGE.np = buf.numpy().view(np.uint32)
    return _STAGE.np


def list_to_device(values, p: int, device) -> torch.Tensor:
    """Python ints -> reduced residues on the device (reference arithmetic
    is mod p throughout, so reducing first is value-preserving)."""
    w = words_from_list(values, p)
    return torch.from_numpy(w.view(np.int32).copy()).to(device, non_blocking=False)


def device_to_list(t: torch.Tensor) -> list[int]:
    return t.to("cpu").contiguous().numpy().view(np.uint32).tolist()


def ptr(t: torch.Tensor) -> int:
    return int(t.data_ptr())
