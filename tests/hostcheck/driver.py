"""Test-only driver: runs the product's replay logic compiled for the host
(libhostcheck.so, see hostcheck.cpp) over numpy buffers laid out exactly as
the device buffers (paper_2512_18725_b200._pack)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from paper_2512_18725_b200 import _abi, _pack

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libhostcheck.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        subprocess.run(["make", "-s", "-C", HERE], check=True)
        L = ctypes.CDLL(SO)
        L.hc_run.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int]
        L.hc_features.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_longlong] + [ctypes.c_void_p] * 3
        L.hc_noise.restype = ctypes.c_double
        L.hc_noise.argtypes = [ctypes.c_ulonglong, ctypes.c_uint, ctypes.c_uint, ctypes.c_double]
        L.hc_noise_k_mismatch.restype = ctypes.c_longlong
        L.hc_noise_k_mismatch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int,
                                          ctypes.c_double]
        for f in ("hc_exp", "hc_log1p"):
            getattr(L, f).restype = ctypes.c_double
            getattr(L, f).argtypes = [ctypes.c_double]
        _lib = L
    return _lib


def run(specs, table: _pack.TableArrays, seg_stride=64, preds=(), noise_k=3):
    pb = _pack.pack(specs, table)
    sz = _pack.sizes(pb, seg_stride, noise_k)
    bufs = {f: np.zeros(sz[k], dtype=dt) for f, dt, k in _pack.BUFFER_PLAN}
    B = _abi.ReplayBuffers()
    for f in _abi.REPLAY_BUFFER_FIELDS:
        setattr(B, f, bufs[f].ctypes.data)
    B.seg_stride, B.cap_max, B.noise_k = seg_stride, pb.cap_max, noise_k
    solo = np.ascontiguousarray(table.solo, dtype=np.float64)
    thr = np.ascontiguousarray(table.thr, dtype=np.float64).reshape(-1)
    T = _abi.Table(solo.ctypes.data, thr.ctypes.data, len(solo), table.max_bs)
    bt = _abi.Batch(ctypes.addressof(pb.scen), ctypes.addressof(pb.models), pb.n_scen, pb.n_models, pb.max_req_cap,
                    max((len(n) for n in pb.names), default=0),
                    max((pb.models[g].list_cap for g in range(pb.n_models)), default=0), 0)
    lib().hc_run(ctypes.byref(bt), ctypes.byref(T), ctypes.byref(B), 1)
    out = {"pb": pb, "bufs": bufs}
    if preds:
        P = (_abi.Predictor * len(preds))(*preds)
        stride = sz["req"]
        X = np.zeros((len(preds), stride, 6))
        Y = np.zeros(stride)
        Yh = np.zeros((len(preds), stride))
        lib().hc_features(ctypes.byref(bt), ctypes.byref(T), ctypes.byref(B), P, len(preds), stride,
                          X.ctypes.data, Y.ctypes.data, Yh.ctypes.data)
        out.update(X=X, Y=Y, Yh=Yh)
    return out


def scenario_view(res, s):
    """Per-scenario arrays in the oracle.run_scenario() key layout."""
    pb, b = res["pb"], res["bufs"]
    S = pb.scen[s]
    ro, n = S.req_off, int(b["n_req"][s])
    nb = int(b["n_batches"][s])
    v = {k: b[k][ro:ro + nb].copy() for k in ("b_model", "b_size", "b_formed", "b_start", "b_completion",
                                                "b_measured", "b_seg_off", "b_nseg")}
    v["order"] = b["out_order"][ro:ro + nb].copy()
    v["r_batch"] = b["r_batch"][ro:ro + n].copy()
    v["arr_t"] = b["arr_t"][ro:ro + n].copy()
    v["arr_model"] = b["arr_model"][ro:ro + n].copy()
    for k in ("s_tbegin", "s_tend", "s_slowdown"):
        v[k] = b[k]
    v["s_colo"] = b["s_colo"].reshape(-1, 3)
    v["status"] = int(b["status"][s])
    v["n_reseats"] = int(b["n_reseats"][s])
    return v
