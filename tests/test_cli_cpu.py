"""CLI front end (mul / sweep over the GPU engines): argument and file
handling that needs no GPU, plus the text format (reference poly.py:184-223,
cli.py exit codes)."""

import pytest

import paper_1609_01010_b200 as mc
from paper_1609_01010_b200 import cli


def _write(path, text):
    path.write_text(text)
    return str(path)


def test_text_round_trip_and_errors():
    fp = mc.FourierPrime.from_modulus(257)
    a = mc.DensePoly(fp, (3, 0, 5, 256))
    assert mc.poly_from_text(mc.poly_to_text(a)) == a
    assert mc.poly_to_text(mc.DensePoly(mc.FourierPrime.from_modulus(17), (3, 0, 5))) == \
        "17\n3\n3 0 5\n"
    assert mc.poly_from_text("17\n0\n\n") == mc.DensePoly.zero(mc.FourierPrime.from_modulus(17))
    for text, line in (("17\n", 2), ("x\n1\n1\n", 1), ("15\n1\n1\n", 1), ("17\nq\n1\n", 2),
                       ("17\n-1\n\n", 2), ("17\n2\n1\n", 3), ("17\n1\nz\n", 3),
                       ("17\n1\n17\n", 3)):
        with pytest.raises(mc.PolyTextError) as e:
            mc.poly_from_text(text)
        assert e.value.line == line, text


def test_mul_exit_codes_without_gpu(tmp_path):
    a = _write(tmp_path / "a.txt", "17\n2\n1 2\n")
    b = _write(tmp_path / "b.txt", "257\n2\n3 4\n")
    bad = _write(tmp_path / "bad.txt", "17\n3\n1 2\n")
    out = str(tmp_path / "c.txt")
    assert cli.main(["mul", a, b, "-o", out]) == cli.EXIT_FIELD_MISMATCH
    assert cli.main(["mul", a, bad, "-o", out]) == cli.EXIT_FILE_FORMAT
    assert cli.main(["mul", a, str(tmp_path / "missing.txt"), "-o", out]) == cli.EXIT_IO


def test_sweep_argument_errors(tmp_path):
    out = str(tmp_path / "s.csv")
    assert cli.main(["sweep", "--min", "4", "--max", "2", "-o", out]) == cli.EXIT_USAGE
    assert cli.main(["sweep", "--min", "1", "--max", "2", "--engines", "fancy", "-o", out]) == \
        cli.EXIT_USAGE
    assert cli.main(["sweep", "--min", "1", "--max", "2", "--step", "0", "-o", out]) == \
        cli.EXIT_USAGE


def test_find_fourier_prime():
    fp = mc.find_fourier_prime(20, 31)
    assert fp.p.bit_length() == 31 and (fp.p - 1) % (1 << 20) == 0
    with pytest.raises(ValueError):
        mc.find_fourier_prime(0, 31)
