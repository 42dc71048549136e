"""ctypes mirror of include/intfsim_b200.h and the loader of the in-tree
sm_100a library `paper_2512_18725_b200/_lib/libintfsim_b200.so`.

There is no CPU implementation behind this module: if the library is missing
the import of any hot-path function raises, and calls without a CUDA device
raise before touching the library.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libintfsim_b200.so")

c_int32 = ctypes.c_int32
c_int64 = ctypes.c_int64
c_double = ctypes.c_double
c_void_p = ctypes.c_void_p
P = ctypes.c_void_p  # every device pointer travels as an address


class Table(ctypes.Structure):
    _fields_ = [("solo_ms", P), ("thr", P), ("n_rows", c_int32), ("max_bs", c_int32)]


class Scenario(ctypes.Structure):
    _fields_ = [
        ("n_models", c_int32), ("model_off", c_int32),
        ("req_off", c_int32), ("req_cap", c_int32),
        ("seg_off", c_int32), ("seg_cap", c_int32),
        ("max_bs", c_int32), ("cap", c_int32),
        ("duration_s", c_double), ("window_ms", c_double), ("sigma", c_double),
        ("beta", c_double * 3),
        ("seed", ctypes.c_uint64), ("oracle_seed", ctypes.c_uint64), ("batch_id_base", ctypes.c_uint64),
    ]


class Model(ctypes.Structure):
    _fields_ = [
        ("entry_base", c_int32), ("name_rank", c_int32), ("crc", ctypes.c_uint32),
        ("list_off", c_int32), ("list_cap", c_int32), ("scen", c_int32),
        ("rate_rps", c_double), ("slo_ms", c_double),
    ]


class Batch(ctypes.Structure):
    _fields_ = [("scen", P), ("models", P), ("n_scen", c_int32), ("n_models", c_int32),
                ("max_req_cap", c_int32), ("max_models", c_int32), ("max_list_cap", c_int32),
                ("req_slots", c_int32), ("long_blocks", P), ("n_long_blocks", c_int32), ("pad_", c_int32)]



REPLAY_BUFFER_FIELDS = [
    "arr_t", "arr_model", "list_t", "list_rid", "n_req", "n_list",
    "b_model", "b_size", "b_formed", "b_start", "b_completion", "b_measured", "b_seg_off", "b_nseg",
    "out_order", "b_running", "r_batch", "r_slo_met",
    "s_tbegin", "s_tend", "s_slowdown", "s_colo",
    "n_batches", "n_segments", "n_reseats", "status", "slot_seg", "noise_tab", "mb_t", "mb_info", "n_mb", "slo_ws",
    "form_ws", "order",
]
SLO_WS_INTS = 256 + 32 * 3 * 256 + 32 * 3 * 4


class ReplayBuffers(ctypes.Structure):
    _fields_ = [(f, P) for f in REPLAY_BUFFER_FIELDS] + [("seg_stride", c_int32), ("cap_max", c_int32),
                                                          ("noise_k", c_int32), ("pad_", c_int32)]


class Jobs(ctypes.Structure):
    _fields_ = [(f, P) for f in ("joff", "jcap", "lo", "hi", "n_jobs", "last", "info", "dirty", "todo",
                                 "todo_count", "slot_scen")] + [("slow", c_double), ("min_len", c_int32),
                                                                ("total_slots", c_int32), ("scratch", P),
                                                                ("own_lo", c_int32), ("own_hi", c_int32)]


class Predictor(ctypes.Structure):
    _fields_ = [("ewma", c_int32), ("pad_", c_int32), ("alpha", c_double), ("w", c_double * 7)]


OLS_WS_DOUBLES = 592 * 35
OLS_FIT_WS_DOUBLES = 128 * 35 + 8

# status bits (INTF_ST_*)
ST_PAST_EVENT, ST_CAP, ST_PROGRESS, ST_NONQUIESCENT, ST_OVERFLOW, ST_SEG_STRIDE = 1, 2, 4, 8, 16, 32

# name -> (restype, argtypes); every symbol include/intfsim_b200.h declares
SIGNATURES = {
    "intf_generate_arrivals": (c_int32, [P, P, P]),
    "intf_split_arrivals": (c_int32, [P, P, P]),
    "intf_replay": (c_int32, [P, P, P, P]),
    "intf_form_batches": (c_int32, [P, P, P]),
    "intf_replay_jobs": (c_int32, [P, P, P, P, P, P, c_int32, P, P, P]),
    "intf_jobs_plan": (c_int32, [P, P, P, P, P]),
    "intf_jobs_replay": (c_int32, [P, P, P, P, c_int32, P]),
    "intf_jobs_verify": (c_int32, [P, P, P, P]),
    "intf_slo_report": (c_int32, [P, P, P, P, P, P, P]),
    "intf_features_predict": (c_int32, [P, P, P, P, c_int32, c_int64, P, P, P, P]),
    "intf_candidate_count": (c_int32, [c_int32, c_int32, P, P, P]),
    "intf_candidate_workspace": (c_int32, [c_int32, c_int32, P]),
    "intf_predict_candidates": (c_int32, [P, c_int32, c_double, P, c_int32, P, P, c_int64, P]),
    "intf_predict_candidates_host": (c_int32, [P, c_int32, c_double, P, c_int32, P, P, c_int64, P]),
    "intf_candidate_prepare": (c_int32, [P, c_int32, c_double, P, c_int64, P]),
    "intf_predict_candidates_prepared": (c_int32, [P, c_int32, P, c_int32, P, P, c_int64, P]),
    "intf_candidate_step": (c_int32, [P, c_int32, c_double, P, c_int32, P, P, P, c_int64, P]),
    "intf_candidate_best_step": (c_int32, [P, c_int32, c_double, P, c_int32, P, P, P, P, c_int64, P]),
    "intf_best_candidates_host": (c_int32, [P, c_int32, c_double, P, c_int32, P, P, c_int64, P]),
    "intf_best_candidates_host_pipelined": (c_int32, [P, c_int32, c_double, P, c_int32, P, P, c_int64, P, P]),
    "intf_best_candidates_host_sync": (c_int32, [P, c_int32, c_double, P, c_int32, P, P, c_int64, P, P]),
    "intf_dispatch_sets": (c_int32, [P, P, c_int32, c_int32, P, P, P]),
    "intf_score_decisions": (c_int32, [P, c_int32, P, P, c_int64, P, P, c_int64, P, P, P]),
    "intf_decision_features_elems": (c_int64, [c_int32, c_int32]),
    "intf_decision_features": (c_int32, [P, c_int32, P, c_int64, P, P]),
    "intf_score_decisions_ft": (c_int32, [P, c_int32, P, P, c_int64, P, P, P, c_int64, P, P, P]),
    "intf_csv_rows": (c_int32, [c_int64, c_int32, P, P, P, P, P, c_int64, P]),
    "intf_repr_f64": (c_int32, [c_double, P, c_int32]),
    "intf_ols_stats": (c_int32, [P, P, c_int64, P, P, P]),
    "intf_ols_solve": (c_int32, [P, P, P, P, P]),
    "intf_ols_fit_rows": (c_int32, [P, P, c_int64, P, P, P, P, P, P]),
    "intf_long_list": (c_int32, []),
    "intf_ols_windows": (c_int32, [P, P, c_int64, c_int32, P, P, P, P]),
    "intf_sgd_streams": (c_int32, [P, P, P, c_int32, P, P, P, P, P]),
    "intf_rls_streams": (c_int32, [P, P, P, c_int32, P, P, P, P, P, P]),
    "intf_eval_report": (c_int32, [P, P, P, c_int32, P, P]),
    "intf_scenario_eval_ws": (c_int64, [c_int32, c_int64]),
    "intf_ols_fit_segments": (c_int32, [P, P, P, P, c_int32, P, P, P, P]),
    "intf_predict_segments": (c_int32, [P, P, P, P, P, c_int32, P, P]),
    "intf_sgd_segments": (c_int32, [P, P, P, P, c_int32, P, P, P, P, P]),
    "intf_rls_segments": (c_int32, [P, P, P, P, c_int32, P, P, P, P, P, P]),
    "intf_eval_segments": (c_int32, [P, P, P, P, c_int32, c_int64, P, P]),
    "intf_scenario_eval": (c_int32, [P, P, P, c_int64, c_int32, c_int32, P, c_double, P, c_int64, P, P, P, P]),
    "intf_features_rows": (c_int32, [P, P, P, P, P, P, c_int64, P, c_int32, P, P, P, P]),
    "intf_predict_rows": (c_int32, [P, c_int64, P, P, P]),
    "intf_quantiles": (c_int32, [P, c_int64, P, c_int32, P, P]),
    "intf_latency_report": (c_int32, [P, P, P, P, c_int64, c_int32, c_double, P, P, P, P]),
    "intf_noise_draws": (c_int32, [ctypes.c_uint64, c_double, P, P, c_int64, P, P]),
    "intf_slowdowns": (c_int32, [P, P, P, P, c_int64, P, P]),
    "intf_scalar": (c_int32, [c_int32, P, c_int32, P, c_int32, P]),
    "intf_rng_stream": (c_int32, [P, c_int32, c_int64, c_int32, P, P]),
    "intf_last_error": (c_int32, [ctypes.c_char_p, c_int32]),
    "intf_abi_version": (c_int32, []),
}

_lib = None


class IntfError(RuntimeError):
    """A C-ABI call returned a non-zero code."""


def load():
    """Load the in-tree CUDA library (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU implementation of the hot path)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib, name, None)
            if f is None:  # reported by tests/test_abi.py; calling it raises AttributeError
                continue
            f.restype = res
            f.argtypes = args
        if lib.intf_abi_version() != 1:
            raise ImportError("libintfsim_b200.so ABI version mismatch")
        _lib = lib
    return _lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(512)
    load().intf_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise IntfError(f"{what} failed (code {rc}): {last_error()}")


def addr(t) -> int:
    """Device (or host) address of a torch tensor / numpy array, or 0."""
    if t is None:
        return 0
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def ref(s):
    return ctypes.cast(ctypes.pointer(s), c_void_p)
