"""PlanSession searches timed on the device (reference tests/test_planner.py
analogues): fresh keys search and grow the store, exact hits do not, the
radix search covers the menu bottom-up and its plans replay bit-correct,
truncated plans mirror into a working inverse, extrapolation past the cap,
and poly_mul(engine="auto") driven by a PlanSession."""

import numpy as np
import pytest
import torch

from conftest import P2

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc
    from paper_1609_01010_b200.plans import PlanKey, PlanSession, PlanStore, plan_mirror


def _session(**kw):
    return PlanSession(PlanStore(), signature="sig", reps=3, **kw)


def test_lookup_searches_once():
    s = _session()
    key = PlanKey("tft", P2, 8, 8, 8, 1)
    e = s.lookup(key)
    assert s.search_count == 1 and len(s.store) == 1 and e.key == key and e.measured_nanos >= 0
    s.lookup(key)
    assert s.search_count == 1


def test_dft_search_menu_bottom_up_and_replay():
    s = _session()
    e = s.search(PlanKey("dft", P2, 8, 0, 8, 1))
    shapes = {(sp, b) for sp, b, _ in s.last_candidates}
    assert ((), 8) in shapes and len(shapes) == 3
    assert e.measured_nanos == min(t for _, _, t in s.last_candidates)
    s.search(PlanKey("dft", P2, 64, 0, 64, 1))
    for L in (2, 4, 8, 16, 32, 64):
        assert s.store.entries_for_key(PlanKey("dft", P2, L, 0, L, 1)), L
    fp = mc.FourierPrime.from_modulus(P2)
    rng = np.random.default_rng(4)
    for entry in s.store:
        x = rng.integers(0, P2, entry.key.L).tolist()
        assert s.replay(entry, x) == mc.moddft(x, mc.get_table(fp, entry.key.L))
    with pytest.raises(mc.UnsupportedSizeError):
        s.search(PlanKey("dft", 17, 64, 0, 64, 1))


def test_truncated_mirror_roundtrip():
    s = _session()
    fwd = s.lookup(PlanKey("tft", P2, 32, 20, 20, 1))
    inv = plan_mirror(fwd)
    s.store.add(inv)
    x = np.random.default_rng(5).integers(0, P2, 20).tolist()
    assert s.replay(inv, s.replay(fwd, x)) == [v * 32 % P2 for v in x]


def test_extrapolation_beyond_cap():
    s = _session(search_cap=16)
    e = s.search(PlanKey("dft", P2, 128, 0, 128, 1))
    capped = s.store.entries_for_key(PlanKey("dft", P2, 16, 0, 16, 1))[0]
    assert e.splits[:3] == (2, 2, 2) and e.splits[3:] == capped.splits
    assert e.base_case == capped.base_case


def test_poly_mul_auto_with_plan_session(tmp_path):
    fp = mc.FourierPrime.from_modulus(P2)
    s = _session()
    rng = np.random.default_rng(6)
    for z1, z2 in ((1, 1), (5, 4), (300, 200), (1500, 2100)):
        a = mc.DensePoly(fp, tuple(rng.integers(1, P2, z1).tolist()))
        b = mc.DensePoly(fp, tuple(rng.integers(1, P2, z2).tolist()))
        got = mc.poly_mul(a, b, mc.ConvRequest(fp, engine="auto", planner=s))
        assert got == mc.poly_mul(a, b, mc.ConvRequest(fp, engine="tft")), (z1, z2)
        assert s.resolve_engine(fp, z1, z2, 1) in ("definition", "fft_pad", "tft")
    path = tmp_path / "store.txt"
    mc.store_save(s.store, str(path))
    assert mc.store_load(str(path)) == s.store
    # a reloaded store under the same signature answers without searching
    s2 = PlanSession(mc.store_load(str(path)), signature="sig")
    s2._mult_nanos.update(s._mult_nanos)
    s2.resolve_engine(fp, 1500, 2100, 1)
    assert s2.search_count == 0
