"""ctypes binding of libmodconv_b200.so (the C ABI in include/modconv_b200.h).

The library is built in-tree by paper_1609_01010_b200/build.py.  There is no
fallback: if the shared library is missing or no CUDA device is present, the
compute entry points raise.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libmodconv_b200.so")

MC_OK, MC_EINVAL, MC_EUNSUPPORTED, MC_ECUDA, MC_ENOMEM = range(5)

_lib = None
_lock = threading.Lock()

u32p = ctypes.c_void_p  # device pointers travel as plain addresses
i32, i64, u32, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
vp = ctypes.c_void_p

_SIGS = {
    "mc_version": ([], ctypes.c_char_p),
    "mc_last_error": ([], ctypes.c_char_p),
    "mc_last_required_two_adicity": ([], ctypes.c_int),
    "mc_launch_count": ([], i64),
    "mc_field_info": ([u32, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(u32)], ctypes.c_int),
    "mc_root_of_unity": ([u32, ctypes.c_int, ctypes.POINTER(u32)], ctypes.c_int),
    "mc_field_prepare": ([u32, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "mc_use_generator": ([u32, u32], ctypes.c_int),
    "mc_conv_fft_pad": ([vp, i64, i32, vp, i64, i32, vp, i64, i64, u32, vp], ctypes.c_int),
    "mc_conv_tft": ([vp, i64, i32, vp, i64, i32, vp, i64, i64, u32, vp], ctypes.c_int),
    "mc_circ_conv": ([vp, vp, vp, i32, i64, u32, vp], ctypes.c_int),
    "mc_conv_direct": ([vp, i64, i32, vp, i64, i32, vp, i64, i64, u32, i32, vp], ctypes.c_int),
    "mc_crt3_slice": ([vp, vp, vp, vp, i64, i64, vp], ctypes.c_int),
    "mc_ipc_alloc": ([i64, ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p], ctypes.c_int),
    "mc_ipc_open": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "mc_ipc_close": ([vp], ctypes.c_int),
    "mc_ipc_free": ([vp], ctypes.c_int),
    "mc_copy_device": ([vp, vp, i64, vp], ctypes.c_int),
    "mc_ntt": ([vp, vp, i32, i64, u32, ctypes.c_int, vp], ctypes.c_int),
    "mc_split_residues": ([vp, vp, vp, i32, i64, u32, vp], ctypes.c_int),
    "mc_recombine_residues": ([vp, vp, vp, i32, i64, u32, vp], ctypes.c_int),
    "mc_nega_conv": ([vp, vp, vp, i32, i64, u32, vp], ctypes.c_int),
    "mc_circ_conv_split": ([vp, vp, vp, i32, i64, u32, vp], ctypes.c_int),
    "mc_tft": ([vp, i32, vp, i32, i32, i64, u32, vp], ctypes.c_int),
    "mc_itft": ([vp, vp, i32, i32, i64, u32, vp], ctypes.c_int),
    "mc_crt3": ([vp, vp, vp, vp, i64, vp], ctypes.c_int),
    "mc_mul_three_primes": ([vp, i32, vp, i32, vp, vp, vp], ctypes.c_int),
    "mc_three_primes_scratch_words": ([i32, i32], i64),
    "mc_mul_mod_prime_k": ([vp, i32, vp, i32, vp, ctypes.c_int, vp], ctypes.c_int),
    "mc_conv_host": ([ctypes.c_int, vp, i64, i32, vp, i64, i32, vp, i64, i64, u32],
                     ctypes.c_int),
    "mc_conv_host_async": ([ctypes.c_int, vp, i64, i32, vp, i64, i32, vp, i64, i64, u32, i64,
                            vp], ctypes.c_int),
    "mc_gen_u32": ([u64, u64, u64, i64, i64, u64, vp, i64, vp], ctypes.c_int),
    "mc_ubench_pass": ([ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "mc_ubench_int_pipes": ([ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                             ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
}

EXPORTED = tuple(_SIGS)


class NativeLibraryMissing(RuntimeError):
    pass


def lib():
    """Load (once) and return the native library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not found; build it with `python -m paper_1609_01010_b200.build`")
            L = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
            _lib = L
    return _lib


def last_error() -> str:
    return lib().mc_last_error().decode()


def check(status: int) -> None:
    """Map a C status to the reference's exception types."""
    if status == MC_OK:
        return
    from .field import UnsupportedSizeError

    msg = last_error()
    if status == MC_EINVAL:
        raise ValueError(msg)
    if status == MC_EUNSUPPORTED:
        req = lib().mc_last_required_two_adicity()
        raise UnsupportedSizeError(msg, required_two_adicity=req if req >= 0 else None)
    if status == MC_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def launch_count() -> int:
    return int(lib().mc_launch_count())
