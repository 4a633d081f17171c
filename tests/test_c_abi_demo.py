"""The drop-in boundary is a plain C ABI: examples/c_abi_demo.c compiles with gcc
against include/moirai_b200.h alone and links the in-tree library.  On CPU it
must report MP_ERR_NO_GPU (no fallback); on a B200 it evaluates all 8
placements of a 3-op chain and agrees with the Python API."""

from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = tmp_path / "c_abi_demo"
    lib = ROOT / "paper_2312_04025_b200"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "c_abi_demo.c"), "-L", str(lib), "-lmoirai_b200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    return exe


def test_c_demo_builds_and_refuses_without_gpu(tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present (covered by the gpu variant)")
    out = subprocess.run([str(_build(tmp_path))], capture_output=True, text=True, check=True).stdout
    assert "no GPU visible" in out and "status -10" in out


@pytest.mark.gpu
def test_c_demo_on_gpu_matches_python(tmp_path):
    import numpy as np

    import paper_2312_04025_b200 as mp

    out = subprocess.run([str(_build(tmp_path))], capture_output=True, text=True, check=True).stdout
    # makespans are printed with %a (exact hexadecimal): compared bit for bit
    got = {line.split()[1]: float.fromhex(line.split()[3]) for line in out.splitlines()
           if line.startswith("placement")}
    c = mp.Cluster([mp.Device(0, 100), mp.Device(1, 100)], {(0, 1): 5e6, (1, 0): 5e6})
    g = mp.CompGraph([mp.OpNode(1, "a", 10, {0: 2.0, 1: 4.0}), mp.OpNode(2, "b", 10, {0: 1.0, 1: 0.5}),
                      mp.OpNode(3, "c", 10, {0: 3.0, 1: 1.0})],
                     [mp.FlowEdge(1, 2, 10_000_000), mp.FlowEdge(2, 3, 20_000_000)])
    rows = np.array([[int(ch) for ch in k] for k in got], dtype=np.uint8)
    ms = mp.evaluate_batch(g, rows, c, mp.effective_bandwidth(c))
    assert [x.hex() for x in ms] == [got[k].hex() for k in got]
    best = next(line for line in out.splitlines() if line.startswith("best row"))
    assert float.fromhex(best.split()[4]) == min(ms)
