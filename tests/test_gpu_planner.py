"""GPU-timed engine selection (engine="auto"): the planner picks one of the
two GPU engines per size class, caches it, persists it atomically, and the
product is the same whichever it picks."""

import json

import numpy as np
import pytest
import torch

from conftest import P2, P3

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc


def test_auto_engine_with_planner(orc, tmp_path):
    store = tmp_path / "plans.json"
    planner = mc.GpuPlanner(batch=64, reps=2, store_path=str(store))
    fp = mc.FourierPrime.from_modulus(P3)
    rng = np.random.default_rng(4)
    for z1, z2 in ((1500, 2100), (2049, 2048), (700, 300)):
        a = rng.integers(1, P3, z1).tolist()
        b = rng.integers(1, P3, z2).tolist()
        req = mc.ConvRequest(fp, engine="auto", planner=planner)
        r = mc.poly_mul(mc.DensePoly(fp, tuple(a)), mc.DensePoly(fp, tuple(b)), req)
        want, _, _ = orc.conv_batch(np.array([a]), np.array([b]), P3)
        assert list(r.coeffs) == want[0].tolist()
    assert planner.search_count == 3
    # cached: no new search
    planner.resolve_engine(fp, 1500, 2100)
    assert planner.search_count == 3
    data = json.loads(store.read_text())
    assert set(data["plans"].values()) <= {"tft", "fft_pad"}
    # a fresh planner reloads the store without searching
    p2 = mc.GpuPlanner(store_path=str(store))
    assert p2.resolve_engine(fp, 1500, 2100) == planner.resolve_engine(fp, 1500, 2100)
    assert p2.search_count == 0


def test_conv_batch_auto(orc):
    a = orc.gen_u32(5, 0, 0, 4, 900, P2)
    b = orc.gen_u32(5, 1, 0, 4, 800, P2)
    at = torch.from_numpy(a.view(np.int32)).cuda()
    bt = torch.from_numpy(b.view(np.int32)).cuda()
    got = mc.conv_batch(at, bt, P2, engine="auto").cpu().numpy().view(np.uint32)
    want, _, _ = orc.conv_batch(a, b, P2)
    assert np.array_equal(got, want)
