"""Build libmoirai_b200.so in-tree with nvcc for sm_100a.

Flags that matter for parity: ``--fmad=false`` (no contraction of the fp64
adds), IEEE division/sqrt (``-prec-div=true``), no fast-math.  ``-lineinfo``
keeps the ncu source page usable.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = PKG / "libmoirai_b200.so"
PEAKS_LIB = PKG / "libmoirai_peaks.so"  # on-chip bandwidth microbenchmarks (bench.py roofline peaks)
OBJ = PKG / "_obj"

SOURCES = ["mp_eval.cu", "mp_instance.cu", "mp_bnb.cu", "mp_aux.cu", "mp_coarsen.cu", "mp_io.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "--fmad=false", "-prec-div=true", "-prec-sqrt=true",
           "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(ROOT / "include")]


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libmoirai_b200")
    return exe


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "moirai_b200.h"]
    srcs = [CSRC / s for s in SOURCES if (CSRC / s).exists()]
    jobs = []
    for src in srcs:
        obj = OBJ / (src.stem + ".o")  # .cpp: host-only translation unit, same nvcc driver
        if force or _stale(obj, [src, *headers]):
            jobs.append([nvcc(), *ARCH, *NVFLAGS, "-c", str(src), "-o", str(obj)])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        return res

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(run, jobs))
    objs = [OBJ / (s.stem + ".o") for s in srcs]
    if force or jobs or _stale(LIB, objs):
        run([nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart_static", "-lrt",
             "-lpthread", "-ldl"])
    psrc = CSRC / "mp_peaks.cu"
    if psrc.exists() and (force or _stale(PEAKS_LIB, [psrc])):
        run([nvcc(), *ARCH, *NVFLAGS, "-shared", "-o", str(PEAKS_LIB), str(psrc), "-lcudart_static", "-lrt",
             "-lpthread", "-ldl"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
