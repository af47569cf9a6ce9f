"""C-ABI argument checking on the GPU box: every compute entry point returns
MC_EINVAL (1) for malformed arguments and MC_EUNSUPPORTED (2) for sizes past
the field's 2-adicity or moduli the 32-bit kernels cannot hold, synchronously
and without launching (mc_launch_count unchanged), with a message in
mc_last_error and, for sizes, the required 2-adicity -- the status codes the
Python layer maps to ValueError / UnsupportedSizeError (field.py:28-33)."""

import ctypes

import pytest
import torch

from conftest import P2, P3

pytestmark = pytest.mark.gpu

EINVAL, EUNSUP = 1, 2

if torch.cuda.is_available():
    from paper_1609_01010_b200 import _native


@pytest.fixture(scope="module")
def env():
    lib = _native.lib()
    buf = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
    return lib, buf.data_ptr(), buf


def _st(lib, rc, want, required=None):
    assert rc == want, (rc, want, lib.mc_last_error())
    if want != 0:
        assert lib.mc_last_error()
    if required is not None:
        assert lib.mc_last_required_two_adicity() == required


def test_conv_entry_points(env):
    lib, d, _ = env
    n0 = lib.mc_launch_count()
    for fn in (lib.mc_conv_fft_pad, lib.mc_conv_tft):
        _st(lib, fn(d, 10, 0, d, 10, 10, d, 20, 1, P2, None), EINVAL)       # empty operand
        _st(lib, fn(d, 5, 10, d, 10, 10, d, 20, 1, P2, None), EINVAL)       # lda < z1
        _st(lib, fn(d, 10, 10, d, 10, 10, d, 18, 1, P2, None), EINVAL)      # ldc < n
        _st(lib, fn(d, 10, 10, d, 10, 10, d, 20, -1, P2, None), EINVAL)     # negative batch
        _st(lib, fn(None, 10, 10, d, 10, 10, d, 20, 1, P2, None), EINVAL)   # null pointer
        _st(lib, fn(d, 10, 10, d, 10, 10, d, 20, 1, 17, None), EUNSUP, 5)   # L = 32 > 2^4
        _st(lib, fn(d, 10, 10, d, 10, 10, d, 20, 1, 2147483659, None), EUNSUP)
        _st(lib, fn(d, 10, 10, d, 10, 10, d, 20, 0, P2, None), 0)           # empty batch: ok
    _st(lib, lib.mc_circ_conv(d, d, d, 24, 1, P2, None), EUNSUP, 24)       # 2-adicity 23
    _st(lib, lib.mc_conv_direct(d, 10, 10, d, 10, 9, d, 10, 1, P2, 1, None), EINVAL)  # circ lengths
    _st(lib, lib.mc_conv_direct(d, 10, 10, d, 10, 10, d, 19, 1, 1, 0, None), EUNSUP)  # modulus 1
    assert lib.mc_launch_count() == n0


def test_transform_entry_points(env):
    lib, d, _ = env
    n0 = lib.mc_launch_count()
    _st(lib, lib.mc_ntt(d, d, 31, 1, P2, 0, None), EINVAL)
    _st(lib, lib.mc_ntt(d, d, 24, 1, P2, 0, None), EUNSUP, 24)
    _st(lib, lib.mc_tft(d, 0, d, 4, 3, 1, P2, None), EINVAL)    # z < 1
    _st(lib, lib.mc_tft(d, 5, d, 4, 3, 1, P2, None), EINVAL)    # z > n
    _st(lib, lib.mc_tft(d, 2, d, 9, 3, 1, P2, None), EINVAL)    # n > L
    _st(lib, lib.mc_itft(d, d, 0, 3, 1, P2, None), EINVAL)      # n < 1
    _st(lib, lib.mc_itft(d, d, 9, 3, 1, P2, None), EINVAL)      # n > L
    _st(lib, lib.mc_itft(d, d, 4, 28, 1, P3, None), EUNSUP, 28)
    assert lib.mc_launch_count() == n0


def test_host_entry_points(env):
    lib, d, _ = env
    a_buf = (ctypes.c_uint32 * 16)(*range(16))
    c = (ctypes.c_uint32 * 32)()
    a, c_ptr = ctypes.addressof(a_buf), ctypes.addressof(c)
    _st(lib, lib.mc_conv_host(2, a, 8, 8, a, 8, 8, c_ptr, 15, 1, P2), EINVAL)  # engine
    _st(lib, lib.mc_conv_host(1, a, 8, 8, a, 8, 8, c_ptr, 15, 1, 17), 0)       # L = 16 fits p = 17
    want = [sum(i * (k - i) for i in range(max(0, k - 7), min(k, 7) + 1)) % 17 for k in range(15)]
    assert list(c)[:15] == want
    _st(lib, lib.mc_conv_host(1, a, 8, 9, a, 8, 8, c_ptr, 16, 1, 17), EINVAL)  # lda < z1
    _st(lib, lib.mc_conv_host(1, a, 16, 16, a, 16, 16, c_ptr, 30, 1, P2), EINVAL)  # ldc < n
