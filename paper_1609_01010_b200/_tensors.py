"""Tensor plumbing between Python containers, torch and the C ABI.

Residues travel as torch.int32 (bit pattern of the uint32 residue; every
residue < 2^31) in contiguous CUDA tensors.  torch is used for device memory
and streams only; all arithmetic happens in the native kernels.
"""

from __future__ import annotations

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


def list_to_device(values, p: int, device) -> torch.Tensor:
    """Python ints -> reduced residues on the device (reference arithmetic
    is mod p throughout, so reducing first is value-preserving)."""
    vals = [int(v) % p for v in values]
    return torch.tensor(vals, dtype=torch.int64).to(torch.int32).to(device, non_blocking=False)


def device_to_list(t: torch.Tensor) -> list[int]:
    return (t.to("cpu").to(torch.int64) & 0xFFFFFFFF).tolist()


def ptr(t: torch.Tensor) -> int:
    return int(t.data_ptr())
