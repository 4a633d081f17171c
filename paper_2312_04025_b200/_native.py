"""ctypes binding of libmoirai_b200.so (the C ABI in include/moirai_b200.h).

There is deliberately no pure-Python or CPU execution path behind these
functions: if the shared library is missing, or no GPU is visible, every call
raises :class:`~paper_2312_04025_b200.errors.NativeError`.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import errors as E

LIB_PATH = Path(__file__).resolve().parent / "libmoirai_b200.so"
# developer override for A/B builds of the same library (never needed in normal use)
if os.environ.get("MOIRAI_B200_LIB"):
    LIB_PATH = Path(os.environ["MOIRAI_B200_LIB"])

MP_OK = 0
MP_ERR_INVALID = -1
MP_ERR_EMPTY_GRAPH = -2
MP_ERR_CYCLE = -3
MP_ERR_MISSING_COST = -4
MP_ERR_TOO_LARGE = -5
MP_ERR_UNSUPPORTED = -6
MP_ERR_CUDA = -7
MP_ERR_MEMORY_EXCEEDED = -8
MP_ERR_BAD_DEVICE = -9
MP_ERR_NO_GPU = -10
MP_ERR_INFEASIBLE_MEMORY = -11

MP_ROW_OK = 0
MP_ROW_MEMORY = 1
MP_ROW_BAD_DEVICE = 2

MP_DEVICE_PTRS = 1

MP_SOLVE_OPTIMAL = 0
MP_SOLVE_FEASIBLE = 1
MP_SOLVE_INFEASIBLE = 2
MP_SOLVE_BUDGET = 3


class mp_error(C.Structure):
    _fields_ = [("code", C.c_int32), ("a", C.c_int64), ("b", C.c_int64), ("msg", C.c_char * 200)]


class mp_problem(C.Structure):
    _fields_ = [
        ("n_ops", C.c_int32), ("n_flows", C.c_int32), ("n_dev", C.c_int32),
        ("cost", C.c_void_p), ("mem", C.c_void_p), ("flow_src", C.c_void_p),
        ("flow_dst", C.c_void_p), ("payload", C.c_void_p), ("cap", C.c_void_p), ("bw", C.c_void_p),
    ]


class mp_instance_info(C.Structure):
    _fields_ = [
        ("n_ops", C.c_int32), ("n_flows", C.c_int32), ("n_dev", C.c_int32),
        ("n_levels", C.c_int32), ("n_sources", C.c_int32), ("ready_cap", C.c_int32),
        ("group_lanes", C.c_int32), ("lanes_used", C.c_int32), ("groups_per_cta", C.c_int32),
        ("ctas", C.c_int32),
        ("smem_bytes", C.c_int32), ("onchip", C.c_int32), ("device", C.c_int32),
        ("n_multi", C.c_int32), ("ready_bound", C.c_int32), ("colo", C.c_int32), ("colo_ok", C.c_int32),
        ("peak_probe", C.c_int32), ("prefilter", C.c_int32), ("mode", C.c_int32),
        ("fastdiv", C.c_int32),
        ("table_bytes", C.c_int64), ("state_bytes", C.c_int64),
        ("tpp_ready_cap", C.c_int32), ("tpp_threads", C.c_int32), ("tpp_kind", C.c_int32),
        ("ls_ready_cap", C.c_int32), ("dur_classes", C.c_int32),
    ]


class mp_violation(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad", C.c_int32), ("x", C.c_int64), ("y", C.c_int64)]


class mp_graph_view(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_edges", C.c_int64), ("n_strings", C.c_int64),
                ("id", C.POINTER(C.c_int64)), ("mem", C.POINTER(C.c_int64)), ("tag", C.POINTER(C.c_int8)),
                ("op_type", C.POINTER(C.c_int32)), ("seq_beg", C.POINTER(C.c_int32)), ("seq", C.POINTER(C.c_int32)),
                ("mem_beg", C.POINTER(C.c_int32)), ("members", C.POINTER(C.c_int64)),
                ("ct_beg", C.POINTER(C.c_int32)), ("ct_dev", C.POINTER(C.c_int64)), ("ct_val", C.POINTER(C.c_double)),
                ("esrc", C.POINTER(C.c_int64)), ("edst", C.POINTER(C.c_int64)), ("epay", C.POINTER(C.c_int64)),
                ("str_beg", C.POINTER(C.c_int64)), ("str", C.c_void_p)]


class mp_coarsen_input(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int32), ("n_edges", C.c_int32), ("n_dev", C.c_int32),
        ("node_id", C.c_void_p), ("seq_beg", C.c_void_p), ("seq_types", C.c_void_p),
        ("tag", C.c_void_p), ("mem", C.c_void_p), ("cost", C.c_void_p),
        ("esrc", C.c_void_p), ("edst", C.c_void_p), ("payload", C.c_void_p),
        ("n_rules", C.c_int32), ("rule_id", C.c_void_p), ("rule_beg", C.c_void_p),
        ("rule_types", C.c_void_p),
        ("n_overrides", C.c_int32), ("ov_beg", C.c_void_p), ("ov_types", C.c_void_p),
        ("ov_dev", C.c_void_p), ("ov_time", C.c_void_p), ("sum_mode", C.c_int32),
    ]


class mp_coarsen_output(C.Structure):
    _fields_ = [
        ("n_groups", C.c_int32), ("n_edges", C.c_int32),
        ("grp_node", C.POINTER(C.c_int32)), ("grp_tag", C.POINTER(C.c_int32)),
        ("mem_beg", C.POINTER(C.c_int32)), ("members", C.POINTER(C.c_int32)),
        ("grp_mem", C.POINTER(C.c_int64)), ("grp_cost", C.POINTER(C.c_double)),
        ("out_src", C.POINTER(C.c_int32)), ("out_dst", C.POINTER(C.c_int32)),
        ("out_payload", C.POINTER(C.c_int64)), ("ordered_replay", C.c_int32),
    ]


# exported symbol -> (restype, argtypes); the exact list include/moirai_b200.h declares
SIGNATURES = {
    "mp_abi_version": (C.c_int32, []),
    "mp_device_count": (C.c_int32, []),
    "mp_launch_count": (C.c_int64, []),
    "mp_instance_create": (C.c_int32, [C.POINTER(mp_problem), C.c_int32, C.POINTER(C.c_void_p),
                                        C.POINTER(mp_error)]),
    "mp_instance_destroy": (None, [C.c_void_p]),
    "mp_instance_info_get": (C.c_int32, [C.c_void_p, C.POINTER(mp_instance_info)]),
    "mp_instance_tune": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint32]),
    "mp_evaluate_batch": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                                       C.POINTER(mp_error)]),
    "mp_evaluate_argmin": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_uint32,
                                        C.c_void_p, C.POINTER(mp_error)]),
    "mp_enumerate_argmin": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_void_p,
                                         C.POINTER(mp_error)]),
    "mp_schedule_one": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.POINTER(C.c_double), C.POINTER(mp_error)]),
    "mp_local_search": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int64,
                                     C.c_int32, C.c_uint64, C.c_void_p, C.POINTER(C.c_double),
                                     C.POINTER(C.c_int64), C.c_void_p, C.c_void_p,
                                     C.POINTER(mp_error)]),
    "mp_branch_and_bound": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_double, C.c_int64, C.c_double,
                                         C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_double),
                                         C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(mp_error)]),
    "mp_greedy_place": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(mp_error)]),
    "mp_audit_schedule": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                       C.c_int64, C.POINTER(C.c_int64), C.POINTER(mp_error)]),
    "mp_graph_load_json": (C.c_int32, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(mp_graph_view),
                                        C.POINTER(mp_error)]),
    "mp_graph_doc_free": (None, [C.c_void_p]),
    "mp_coarsen": (C.c_int32, [C.POINTER(mp_coarsen_input), C.c_int32, C.POINTER(mp_coarsen_output),
                               C.POINTER(mp_error)]),
    "mp_coarsen_free": (None, [C.POINTER(mp_coarsen_output)]),
}

_lib = None


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load (once) and type the shared library; raise NativeError if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise E.NativeError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def lib() -> C.CDLL:
    return load_library()


def ptr(a: np.ndarray | None):
    return None if a is None else C.c_void_p(a.ctypes.data)


def check(code: int, err: mp_error, context: str = "") -> None:
    """Map an MP_ERR_* status onto the reference exception tree."""
    if code == MP_OK:
        return
    msg = err.msg.decode(errors="replace")
    if code == MP_ERR_EMPTY_GRAPH:
        raise ValueError("cannot place an empty graph")
    if code == MP_ERR_TOO_LARGE:
        raise E.TooLargeError(int(err.a), int(err.b))
    if code == MP_ERR_INVALID:
        raise ValueError(f"{context}: {msg}")
    if code == MP_ERR_INFEASIBLE_MEMORY:
        raise E.InfeasibleMemoryError(int(err.a), int(err.b))
    if code == MP_ERR_BAD_DEVICE:
        raise KeyError(f"{context}: {msg}")
    raise E.NativeError(f"{context}: status {code}: {msg}")


def require_gpu() -> None:
    n = lib().mp_device_count()
    if n <= 0:
        raise E.NativeError("no CUDA device visible; libmoirai_b200 has no CPU fallback")
