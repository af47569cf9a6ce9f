"""The reference-side binding of INTEGRATION.md, exercised as written: plain
ctypes on libmodconv_b200.so with array.array buffers (pageable host memory,
no torch), mc_conv_host for both north-star engines, UnsupportedSizeError
mapping through mc_last_required_two_adicity."""

import array
import ctypes

import numpy as np
import pytest

from conftest import P1, P2, P3

pytestmark = pytest.mark.gpu


class UnsupportedSizeError(ValueError):
    def __init__(self, msg, required):
        super().__init__(msg)
        self.required_two_adicity = required


def _lib():
    from paper_1609_01010_b200._native import LIB_PATH

    lib = ctypes.CDLL(LIB_PATH)
    lib.mc_conv_host.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                 ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                 ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32]
    lib.mc_last_error.restype = ctypes.c_char_p
    lib.mc_last_required_two_adicity.restype = ctypes.c_int
    return lib


def gpu_linear_conv(lib, u, v, p, engine):  # the INTEGRATION.md stub
    n = len(u) + len(v) - 1
    a = array.array("I", (x % p for x in u))
    b = array.array("I", (x % p for x in v))
    c = array.array("I", bytes(4 * n))
    st = lib.mc_conv_host(engine, a.buffer_info()[0], len(a), len(a), b.buffer_info()[0], len(b),
                          len(b), c.buffer_info()[0], n, 1, p)
    if st == 2:
        req = lib.mc_last_required_two_adicity()
        raise UnsupportedSizeError(lib.mc_last_error().decode(), req if req >= 0 else None)
    if st != 0:
        raise ValueError(lib.mc_last_error().decode())
    return c.tolist()


@pytest.mark.parametrize("p", [17, P1, P2, P3])
def test_stub_matches_oracle(orc, p):
    lib = _lib()
    for z1, z2 in ((1, 1), (2, 2), (300, 17), (1500, 2100), (5000, 4000), (20000, 9000)):
        u = orc.gen_u32(80, 0, z1, 1, z1, p)[0]
        v = orc.gen_u32(80, 1, z2, 1, z2, p)[0]
        if p == 17 and z1 + z2 - 1 > 16:
            continue  # 2-adicity 4
        want, _, _ = orc.conv_batch(u[None], v[None], p)
        for engine in (0, 1):
            got = gpu_linear_conv(lib, u.tolist(), v.tolist(), p, engine)
            assert np.array_equal(np.array(got, dtype=np.uint32), want[0]), (p, z1, z2, engine)


def test_stub_reference_kats():
    lib = _lib()
    assert gpu_linear_conv(lib, [1, 2], [3, 4], 17, 0) == [3, 10, 8]   # test_convolve.py:109-115
    assert gpu_linear_conv(lib, [1, 2], [3, 4], 17, 1) == [3, 10, 8]   # test_convolve.py:209-212
    assert gpu_linear_conv(lib, [5], [7], 17, 1) == [1]


def test_stub_unsupported_size():
    lib = _lib()
    with pytest.raises(UnsupportedSizeError) as ei:
        gpu_linear_conv(lib, [1] * 20, [1] * 20, 17, 0)  # L = 64 > 2^4
    assert ei.value.required_two_adicity == 6
    assert lib.mc_conv_host(2, None, 1, 1, None, 1, 1, None, 1, 1, 17) == 1  # MC_EINVAL: engine
