"""The product path never touches the oracle: no module of the package (or
its CUDA sources) imports, links or loads anything under oracle/, importing
the package does not pull the oracle in, and every compute entry point
raises when the CUDA library or a device is missing instead of falling back
to the CPU."""

import ast
import os
import subprocess
import sys

import pytest

from conftest import REPO

PKG = os.path.join(REPO, "paper_1609_01010_b200")


def test_no_oracle_imports_in_package():
    for name in os.listdir(PKG):
        if not name.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(PKG, name)).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                mods = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                mods = [node.module or ""]
            else:
                continue
            assert not any(m.split(".")[0] == "oracle" for m in mods), (name, mods)
        src = open(os.path.join(PKG, name)).read()
        assert "modconv_oracle" not in src and "liboracle" not in src, name
    for name in os.listdir(os.path.join(PKG, "csrc")):
        src = open(os.path.join(PKG, "csrc", name)).read()
        assert "#include" not in src or "oracle" not in "".join(
            l for l in src.splitlines() if l.startswith("#include")), name


def test_import_does_not_load_oracle():
    code = ("import sys; import paper_1609_01010_b200 as mc; "
            "print(any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules))")
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, capture_output=True, text=True,
                         check=True).stdout.strip()
    assert out == "False"


def test_compute_paths_fail_loudly_without_a_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("this container check needs a CPU-only host")
    import paper_1609_01010_b200 as mc

    fp = mc.FourierPrime.from_modulus(998244353)
    a = mc.DensePoly(fp, (1, 2))
    for engine in ("tft", "fft_pad", "definition", "split"):
        with pytest.raises(Exception) as err:
            mc.poly_mul(a, a, mc.ConvRequest(fp, engine=engine))
        assert "CUDA" in str(err.value) or "cuda" in str(err.value) or "device" in str(err.value)
    with pytest.raises(Exception):
        mc.conv_batch(torch.ones((1, 4), dtype=torch.int32), torch.ones((1, 4), dtype=torch.int32),
                      998244353)
    with pytest.raises(Exception):
        mc.lin_conv_def([1, 2], [3], fp)
