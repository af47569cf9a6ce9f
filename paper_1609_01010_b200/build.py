"""Build libmodconv_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_1609_01010_b200.build          # incremental
    python -m paper_1609_01010_b200.build --clean

Every .cu under csrc/ becomes one object (conv_small_inst.cu once per
transform size K = 4..13, so the heavily unrolled kernels compile in
parallel); the objects are linked into paper_1609_01010_b200/_lib/.
"""

from __future__ import annotations

import argparse
import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib")
OBJ = os.path.join(OUT, "obj")
LIB = os.path.join(OUT, "libmodconv_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-Wall", f"-I{INCLUDE}", f"-I{CSRC}"]
SMALL_KS = range(4, 14)
COL_KRS = range(4, 14)


def _units():
    units = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        base = os.path.splitext(os.path.basename(src))[0]
        if base == "conv_small_inst":
            for k in SMALL_KS:
                units.append((src, os.path.join(OBJ, f"{base}_k{k}.o"), [f"-DMC_K={k}"]))
        elif base == "fourstep_cols":
            for k in COL_KRS:
                units.append((src, os.path.join(OBJ, f"{base}_kr{k}.o"), [f"-DMC_KR={k}"]))
        else:
            units.append((src, os.path.join(OBJ, base + ".o"), []))
    return units


def _deps_mtime():
    files = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    files += glob.glob(os.path.join(INCLUDE, "*.h"))
    return max((os.path.getmtime(f) for f in files), default=0.0)


def _compile(unit, verbose):
    src, obj, extra = unit
    cmd = [NVCC, *ARCH, *FLAGS, *extra, *os.environ.get("MC_EXTRA_FLAGS", "").split(), "-c",
           src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src} {extra}:\n{r.stderr}")
    return (obj, r.stderr if verbose else "")


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    dep = _deps_mtime()
    stamp = os.path.join(OBJ, "extra_flags.txt")  # MC_EXTRA_FLAGS of the objects on disk
    extra_now = os.environ.get("MC_EXTRA_FLAGS", "").strip()
    try:
        with open(stamp) as f:
            force = force or f.read() != extra_now
    except OSError:
        force = True
    with open(stamp, "w") as f:
        f.write(extra_now)
    todo = []
    units = _units()
    for u in units:
        src, obj, _ = u
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(
                os.path.getmtime(src), dep):
            todo.append(u)
    if todo:
        jobs = jobs or min(len(todo), os.cpu_count() or 4)
        with ThreadPoolExecutor(jobs) as ex:
            for obj, log in ex.map(lambda u: _compile(u, verbose), todo):
                if verbose and log:
                    print(log, file=sys.stderr)
    objs = [u[1] for u in units]
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(o) for o in objs):
        tmp = LIB + ".tmp"
        subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs], check=True)
        os.replace(tmp, LIB)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    args = ap.parse_args()
    if args.clean:
        shutil.rmtree(OUT, ignore_errors=True)
        return
    print(build(force=args.force, verbose=args.verbose))


if __name__ == "__main__":
    main()
