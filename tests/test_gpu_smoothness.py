"""The reference's machine-local timing criterion (pkg/tests/test_acceptance.py:197-235,
`test_criterion_6_smoothness_timing`, marked slow there) on the B200, with
device time: just past each power of two the truncated engine is faster than
the padded one, and its boundary-crossing ratio stays far below the padded
engine's jump.  Batched calls of ~2^24 product positions (launch latency does
not count), CUDA events, median of the repetitions; products checked equal
between the two engines."""

import statistics

import pytest
import torch

from conftest import P2

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc
    from gpu_helpers import gen_device


def _median_ms(fn, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


@pytest.mark.parametrize("k", [11, 12, 13, 14, 15, 16])
def test_criterion_6_smoothness_timing_device(k):
    fp = mc.FourierPrime.from_modulus(P2)

    def inputs(total, seed):
        z1 = (total + 1) // 2
        z2 = total + 1 - z1
        rows = max(8, (1 << 24) >> (k + 1))
        return (gen_device(seed, 0, 0, rows, z1, P2), gen_device(seed, 1, 0, rows, z2, P2))

    at_pow = inputs(1 << k, 60 + k)
    past_pow = inputs((1 << k) + 1, 80 + k)
    t = {}
    outs = {}
    for engine in ("tft", "fft_pad"):
        for tag, (a, b) in (("past", past_pow), ("at", at_pow)):
            out = mc.conv_batch(a, b, fp, engine=engine)
            t[engine, tag] = _median_ms(lambda: mc.conv_batch(a, b, fp, engine=engine, out=out))
            outs[engine, tag] = out
    for tag in ("past", "at"):
        assert torch.equal(outs["tft", tag], outs["fft_pad", tag])
    assert t["tft", "past"] < t["fft_pad", "past"], (k, t)
    tft_ratio = t["tft", "past"] / t["tft", "at"]
    fft_ratio = t["fft_pad", "past"] / t["fft_pad", "at"]
    assert tft_ratio <= 0.5 * fft_ratio + 1, (k, tft_ratio, fft_ratio)
