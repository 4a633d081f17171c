"""The C ABI library loads, exports exactly what include/moirai_b200.h declares,
and — with no GPU visible — refuses to compute instead of falling back to CPU."""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2312_04025_b200 as mp
from paper_2312_04025_b200 import _native as N

HEADER = Path(__file__).resolve().parents[1] / "include" / "moirai_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mp_[a-z_]+)\s*\(", text)))


def test_header_declares_what_the_binding_types():
    assert declared_symbols() == sorted(N.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(N.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.mp_abi_version() == 1


def test_struct_layouts_match_header():
    # spot-check sizes against the header's field lists
    assert C.sizeof(N.mp_error) == 8 + 8 + 8 + 200  # int32 padded to 8, two int64, char[200]
    assert C.sizeof(N.mp_problem) == 16 + 7 * 8
    # 21 int32 (+ pad) + 2 int64 + 5 int32 (tpp_ready_cap, tpp_threads, tpp_kind, ls_ready_cap,
    # dur_classes) + pad
    assert C.sizeof(N.mp_instance_info) == 22 * 4 + 2 * 8 + 6 * 4
    assert C.sizeof(N.mp_violation) == 4 + 4 + 8 + 8
    assert C.sizeof(N.mp_graph_view) == 3 * 8 + 16 * 8


def _no_gpu():
    return N.lib().mp_device_count() == 0


@pytest.mark.skipif(not _no_gpu(), reason="only meaningful where no GPU is visible")
def test_no_cpu_fallback_without_gpu():
    g = mp.CompGraph([mp.OpNode(1, "conv", 1, {0: 1.0, 1: 2.0})], [])
    c = mp.Cluster([mp.Device(0, 10), mp.Device(1, 10)], {(0, 1): 1e6, (1, 0): 1e6})
    with pytest.raises(mp.NativeError):
        mp.schedule_for_assignment(g, c, mp.effective_bandwidth(c), {1: 0})
    with pytest.raises(mp.NativeError):
        mp.gcof(g, mp.FusionRuleSet([]))


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(mp.NativeError):
        N.load_library(tmp_path / "nope.so")


def test_validation_before_the_gpu():
    """Errors the reference raises before any scheduling are raised host-side
    in the same order (solver.py:46-55)."""
    c = mp.Cluster([mp.Device(0, 10), mp.Device(1, 10)], {(0, 1): 1e6, (1, 0): 1e6})
    mesh = mp.effective_bandwidth(c)
    with pytest.raises(ValueError):
        mp.Instance(mp.CompGraph([], []), c, mesh)
    with pytest.raises(mp.MissingCostError) as ei:
        mp.Instance(mp.CompGraph([mp.OpNode(1, "conv", 1, {0: 1.0})], []), c, mesh)
    assert (ei.value.op, ei.value.device) == (1, 1)
    assert np.isnan(np.nan)


def test_departures_raise_clear_errors_before_the_gpu():
    """Documented departures of the drop-in surface: more than
    16 devices -> DeviceLimitError; a NaN cost -> ValueError (not MissingCostError,
    which the reference reserves for absent entries)."""
    devs = [mp.Device(k, 10) for k in range(17)]
    c17 = mp.Cluster(devs, {(a, b): 1e6 for a in range(17) for b in range(17) if a != b})
    g = mp.CompGraph([mp.OpNode(1, "conv", 1, {k: 1.0 for k in range(17)})], [])
    with pytest.raises(mp.DeviceLimitError) as ei:
        mp.Instance(g, c17, mp.effective_bandwidth(c17))
    assert (ei.value.devices, ei.value.limit) == (17, 16)
    assert isinstance(ei.value, mp.NativeError)
    c = mp.Cluster([mp.Device(0, 10), mp.Device(1, 10)], {(0, 1): 1e6, (1, 0): 1e6})
    with pytest.raises(ValueError, match="NaN"):
        mp.Instance(mp.CompGraph([mp.OpNode(1, "conv", 1, {0: float("nan"), 1: 1.0})], []), c,
                    mp.effective_bandwidth(c))


def test_check_feasibility_of_an_empty_graph_is_empty():
    """The reference's audit loops are empty for an empty graph (simulator.py:179-264)."""
    c = mp.Cluster([mp.Device(0, 10), mp.Device(1, 10)], {(0, 1): 1e6, (1, 0): 1e6})
    s = mp.Schedule({}, {}, {}, {}, 0.0)
    assert mp.check_feasibility(s, mp.CompGraph([], []), c, mp.effective_bandwidth(c)) == []


def test_non_uint8_rows_are_range_checked():
    """int rows are not cast modulo 256 onto valid device indices."""
    from paper_2312_04025_b200.solver import _rows

    class _Inst:
        n_ops, K = 3, 4

    with pytest.raises(ValueError):
        _rows(_Inst(), np.array([[0, 1, 260]], dtype=np.int64))
    with pytest.raises(ValueError):
        _rows(_Inst(), np.array([[0, -1, 2]], dtype=np.int32))
    with pytest.raises(ValueError):
        _rows(_Inst(), np.array([[0.0, 1.0, 2.0]]))
    assert _rows(_Inst(), np.array([[0, 1, 3]], dtype=np.int64)).dtype == np.uint8
