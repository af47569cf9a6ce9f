"""Plan records, the modconv-plan v1 store format and the session's lookup /
engine-choice policy (reference tests/test_planner.py analogues) -- the
host-side parts, no kernel timed."""

import random

import pytest

from paper_1609_01010_b200 import FourierPrime, plans
from paper_1609_01010_b200.plans import (STORE_VERSION, PlanEntry, PlanFormatError, PlanKey,
                                         PlanSession, PlanStore, make_exec_signature, plan_mirror,
                                         store_load, store_save)

P = 998244353


def test_key_ordering_and_validation():
    keys = [PlanKey(k, p, L, 0, L, t) for k in ("tft", "dft") for p in (257, 17)
            for L in (8, 4) for t in (2, 1)]
    assert sorted(keys)[0] == PlanKey("dft", 17, 4, 0, 4, 1)
    for bad in (("fft", 17, 8, 0, 8, 1), ("dft", 17, 6, 0, 6, 1), ("dft", 17, 8, 0, 8, 0),
                ("dft", 17, 8, -1, 8, 1)):
        with pytest.raises(ValueError):
            PlanKey(*bad)


def test_entry_validation_and_mirror():
    k = PlanKey("tft", 17, 64, 20, 40, 1)
    e = PlanEntry(k, (2, 4), 8, 10, "sig")
    m = plan_mirror(e)
    assert m.key.kind == "itft" and m.splits == (4, 2) and m.base_case == 8
    assert plan_mirror(m) == e
    with pytest.raises(ValueError):
        plan_mirror(PlanEntry(PlanKey("dft", 17, 8, 0, 8, 1), (), 8, 1, "s"))
    for splits, base, nanos, sig in (((3,), 8, 1, "s"), ((2,), 8, 1, "s"), ((2, 4), 8, -1, "s"),
                                     ((2, 4), 8, 1, "a|b"), ((2, 4), 16, 1, "s")):
        with pytest.raises(ValueError):
            PlanEntry(k, splits, base, nanos, sig)


def test_store_format(tmp_path):
    path = tmp_path / "plans.txt"
    store_save(PlanStore(), str(path))
    assert path.read_text() == f"{STORE_VERSION}\n"
    assert store_load(str(path)) == PlanStore()
    store = PlanStore()
    store.add(PlanEntry(PlanKey("dft", 17, 8, 0, 8, 1), (2,), 4, 55, "sig"))
    store_save(store, str(path))
    lines = path.read_text().splitlines()
    assert lines == [STORE_VERSION, "dft|17|8|0|8|1|splits=2|base=4|nanos=55|sig=sig"]
    with pytest.raises(ValueError):
        store.add(PlanEntry(PlanKey("dft", 17, 8, 0, 8, 1), (2,), 4, 55, "sig"))
    path.write_text("modconv-plan v0\n")
    with pytest.raises(PlanFormatError) as err:
        store_load(str(path))
    assert err.value.line == 1
    path.write_text(f"{STORE_VERSION}\ndft|17|8|0|8|1|splits=2|base=4|nanos=55|sig=s\n"
                    "dft|17|8|0|8|1|splits=2|base=4|nanos=x|sig=s\n")
    with pytest.raises(PlanFormatError) as err:
        store_load(str(path))
    assert err.value.line == 3


def test_store_fuzzed_round_trips(tmp_path):
    rng = random.Random(7)
    path = tmp_path / "f.txt"
    for trial in range(30):
        store = PlanStore()
        for _ in range(rng.randrange(0, 8)):
            lg = rng.randrange(1, 12)
            L = 1 << lg
            kind = rng.choice(("dft", "tft", "itft", "conv"))
            n = rng.randrange(0, L + 1)
            key = PlanKey(kind, rng.choice((17, 257, P)), L, rng.randrange(0, n + 1), n,
                          rng.randrange(1, 5))
            splits, size = [], L
            while size > 8 or (size > 1 and rng.random() < 0.5 and size not in (2, 4, 8)):
                r = rng.choice([r for r in (2, 4, 8) if size % r == 0 and size // r >= 2])
                splits.append(r)
                size //= r
            if size == 1:
                continue
            store.add(PlanEntry(key, tuple(splits), size, rng.randrange(0, 10**9),
                                f"host-{rng.randrange(3)};cores=8"), replace_existing=True)
        store_save(store, str(path))
        assert store_load(str(path)) == store, trial


def _session(store=None, sig="this-host"):
    return PlanSession(store or PlanStore(), signature=sig, reps=2)


def test_signature_miss_clones_without_search():
    store = PlanStore()
    original = PlanEntry(PlanKey("dft", 17, 8, 0, 8, 1), (2,), 4, 55, "other-host")
    store.add(original)
    s = _session(store)
    clone = s.lookup(original.key)
    assert s.search_count == 0 and clone.exec_signature == "this-host"
    assert clone.splits == original.splits and len(store) == 2
    assert store.get(original.key, "other-host") == original
    with pytest.raises(ValueError):
        s.search(PlanKey("conv", 17, 8, 0, 8, 1))


def _stocked(tft_ns, dft_ns, mult_ns=50.0):
    s = _session()
    for z in (8, 9, 15, 16):
        s.store.add(PlanEntry(PlanKey("tft", P, 16, z, 15, 1), (2, 2, 2), 2, tft_ns, s.signature))
    s.store.add(PlanEntry(PlanKey("itft", P, 16, 15, 15, 1), (2, 2, 2), 2, tft_ns, s.signature))
    s.store.add(PlanEntry(PlanKey("dft", P, 16, 0, 16, 1), (2, 2), 4, dft_ns, s.signature))
    s._mult_nanos[P] = mult_ns
    return s


def test_resolve_engine_policy():
    fp = FourierPrime.from_modulus(P)
    assert _stocked(10, 1000).resolve_engine(fp, 8, 8, 1) == "tft"
    assert _stocked(10**6, 10).resolve_engine(fp, 8, 8, 1) == "fft_pad"
    assert _stocked(10**6, 10**6).resolve_engine(fp, 8, 8, 1) == "definition"
    assert _session().resolve_engine(fp, 1, 1, 1) == "definition"
    assert _session().resolve_engine(FourierPrime.from_modulus(7), 5, 5, 1) == "definition"
    assert _session().resolve_engine(FourierPrime.from_modulus(17), 10, 10, 1) == "definition"


def test_exec_signature():
    sig = make_exec_signature(3)
    assert "threads=3" in sig and "cores=" in sig and "build=modconv-" in sig
    assert "|" not in sig and "\n" not in sig
    assert make_exec_signature(2) == make_exec_signature(2)
    assert plans.STORE_VERSION == "modconv-plan v1"
