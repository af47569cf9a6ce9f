"""CLI mul / sweep on the GPU (reference tests/test_cli.py analogues)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1609_01010_b200 as mc
    from paper_1609_01010_b200 import cli


def test_mul_each_engine(tmp_path, orc):
    a = tmp_path / "a.txt"
    b = tmp_path / "b.txt"
    a.write_text("998244353\n5\n1 2 3 4 5\n")
    b.write_text("998244353\n3\n7 0 998244352\n")
    want = orc.schoolbook([1, 2, 3, 4, 5], [7, 0, 998244352], 998244353)
    for engine in ("fft_pad", "tft", "split", "definition", "auto"):
        out = tmp_path / f"c_{engine}.txt"
        assert cli.main(["mul", str(a), str(b), "--engine", engine, "-o", str(out)]) == 0
        c = mc.poly_from_text(out.read_text())
        assert list(c.coeffs) == want, engine


def test_mul_unsupported_size(tmp_path):
    a = tmp_path / "a.txt"
    a.write_text("17\n10\n" + " ".join(["1"] * 10) + "\n")
    assert cli.main(["mul", str(a), str(a), "--engine", "tft", "-o",
                     str(tmp_path / "c.txt")]) == cli.EXIT_UNSUPPORTED


def test_sweep_schema_counters_and_sentinels(tmp_path):
    out = tmp_path / "s.csv"
    assert cli.main(["sweep", "--min", "7", "--max", "10", "--engines", "fft_pad,tft",
                     "--reps", "3", "-o", str(out)]) == 0
    rows = out.read_text().splitlines()
    assert rows[0] == cli.HEADER
    assert len(rows) == 1 + 4 * 2
    by = {(r.split(",")[0], r.split(",")[1]): r.split(",") for r in rows[1:]}
    # n = 9: fft_pad pads to 16 -> 3*8*4 butterflies, 16 pointwise; tft: n pointwise
    assert by[("9", "fft_pad")][5:] == ["96", "16"]
    assert by[("9", "tft")][6] == "9"
    # 17 has 2-adicity 4: sizes needing L = 32 get the sentinel row
    out2 = tmp_path / "s2.csv"
    assert cli.main(["sweep", "--min", "15", "--max", "17", "--prime", "17", "--reps", "2",
                     "-o", str(out2)]) == 0
    rows2 = out2.read_text().splitlines()[1:]
    assert any(r.endswith(",-1,-1,-1,-1") for r in rows2)
    out3 = tmp_path / "s3.csv"
    assert cli.main(["sweep", "--min", "3000", "--max", "3001", "--batch", "64", "--reps", "2",
                     "-o", str(out3)]) == 0


def test_sweep_definition_rows_beyond_two_adicity(tmp_path):
    """Definition (and auto) rows keep working at every size (reference
    tests/test_cli.py:171-178): p = 17 has no transform past length 16."""
    out = tmp_path / "d.csv"
    assert cli.main(["sweep", "--min", "15", "--max", "20", "--engines", "tft,definition,auto",
                     "--prime", "17", "--reps", "2", "-o", str(out)]) == 0
    by = {(r.split(",")[0], r.split(",")[1]): r.split(",") for r in
          out.read_text().splitlines()[1:]}
    assert by[("20", "tft")][3] == "-1"
    for n in range(15, 21):
        assert by[(str(n), "definition")][3] != "-1"
        assert by[(str(n), "auto")][3] != "-1"
    assert by[("20", "definition")][5:] == ["0", "0"]


def test_plan_and_mul_auto_store(tmp_path):
    """`plan` writes a modconv-plan v1 store (dft/tft planned, itft mirrored);
    `mul --engine auto --store` reuses and extends it (cli.py:95-171)."""
    store = tmp_path / "plans.txt"
    assert cli.main(["plan", "--store", str(store), "--max-l", "64"]) == 0
    st = mc.store_load(str(store))
    assert len(st) == 3 * 6
    kinds = sorted({e.key.kind for e in st})
    assert kinds == ["dft", "itft", "tft"]
    assert cli.main(["plan", "--store", str(store), "--max-l", "48"]) == cli.EXIT_USAGE
    assert cli.main(["plan", "--store", str(store), "--max-l", "64", "--prime", "17"]) == \
        cli.EXIT_UNSUPPORTED
    a = tmp_path / "a.txt"
    a.write_text("998244353\n5\n1 2 3 4 5\n")
    out = tmp_path / "c.txt"
    assert cli.main(["mul", str(a), str(a), "--store", str(store), "-o", str(out)]) == 0
    assert mc.poly_from_text(out.read_text()).coeffs == (1, 4, 10, 20, 35, 44, 46, 40, 25)
    assert len(mc.store_load(str(store))) >= len(st)
    bad = tmp_path / "bad.txt"
    bad.write_text("not a store\n")
    assert cli.main(["mul", str(a), str(a), "--store", str(bad), "-o", str(out)]) == \
        cli.EXIT_FILE_FORMAT
