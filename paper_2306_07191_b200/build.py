"""In-tree build of libnif_b200.so (sm_100a) and the CPU oracle library.

    python -m paper_2306_07191_b200.build

Exact-arithmetic translation units (fp64 geometry, reference-exact encode
and dense forward) are compiled with -fmad=false so no multiply-add is
contracted; the tensor-core and training units use the default.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
EXACT_UNITS = ["trace.cu", "exact.cu", "gather.cu", "train.cu", "sah_gpu.cu"]
FAST_UNITS = ["query.cu"]
HOST_UNITS = ["sah_builder.cpp", "api.cpp", "engine.cpp"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def build(verbose: bool = False) -> Path:
    nvcc = _nvcc()
    BUILD.mkdir(exist_ok=True)
    inc = ["-I", str(ROOT / "include"), "-I", str(CSRC)]
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off",
              "--expt-relaxed-constexpr"] + inc
    objs = []
    for unit in EXACT_UNITS + FAST_UNITS:
        src = CSRC / unit
        if not src.exists():
            continue
        obj = BUILD / (unit + ".o")
        flags = ["-fmad=false"] if unit in EXACT_UNITS else []
        extra = ["-Xptxas", "-v"] if verbose else []
        r = _run([nvcc, *ARCH, *common, *flags, *extra, "-c", str(src), "-o", str(obj)])
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(str(obj))
    for unit in HOST_UNITS:
        obj = BUILD / (unit + ".o")
        _run([nvcc, *common, "-x", "cu", "-c", str(CSRC / unit), "-o", str(obj)]
             if unit.endswith(".cu") else
             ["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off",
              "-I", str(ROOT / "include"), "-I", str(CSRC), "-I", "/usr/local/cuda/include",
              "-c", str(CSRC / unit), "-o", str(obj)])
        objs.append(str(obj))
    out = PKG / "libnif_b200.so"
    tmp = PKG / "libnif_b200.so.tmp"
    _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs,
          "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"])
    os.replace(tmp, out)
    return out


def build_oracle() -> Path:
    """CPU restatement used only by tests / bench's cpu_baseline leg."""
    src = ROOT / "oracle" / "nif_oracle.c"
    out = ROOT / "oracle" / "liboracle.so"
    _run(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
          "-fopenmp", "-o", str(out), str(src), "-lm"])
    return out


if __name__ == "__main__":
    p = build(verbose="-v" in sys.argv)
    print(p)
    if (ROOT / "oracle" / "nif_oracle.c").exists():
        print(build_oracle())
