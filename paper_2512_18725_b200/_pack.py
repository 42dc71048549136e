"""Pack scenarios and a profile table into the C-ABI descriptor arrays.

Host-side layout planning only (no simulation math): capacities, offsets and
the per-model metadata the kernels need (table rows, crc32 keys
`profiles.py:239-243`, string-order ranks used by the (t, model_id) arrival
sort `workload.py:96`).

Scenario inputs are the reference's JSON scenario dict (`workload.py:192-218`
`scenario_to_dict` layout); `TableArrays` is the flattened profile table.
"""
from __future__ import annotations

import math
import zlib
from dataclasses import dataclass, field

import numpy as np

from . import _abi


@dataclass
class TableArrays:
    """Profile table as SoA fp64: row = model_index * max_bs + (bs - 1)."""

    models: list
    max_bs: int
    solo: np.ndarray  # [rows]
    thr: np.ndarray  # [rows, 3] (l2, dram, sm)
    missing: frozenset = frozenset()  # rows with no profile entry (zero-filled; a batch there is a ProfileError)

    def row(self, model_id: str, bs: int) -> int:
        return self.models.index(model_id) * self.max_bs + bs - 1

    @property
    def n_rows(self) -> int:
        return len(self.solo)


@dataclass
class PackedBatch:
    specs: list
    table: TableArrays
    scen: object  # ctypes array of _abi.Scenario
    models: object  # ctypes array of _abi.Model
    names: list = field(default_factory=list)  # per scenario: deployed model ids
    n_scen: int = 0
    n_models: int = 0
    total_req: int = 0
    total_list: int = 0
    total_seg: int = 0
    max_req_cap: int = 0
    cap_max: int = 1


def _list_capacity(rate: float, duration_s: float, scale: float) -> int:
    if rate <= 0:
        return 0
    mu = rate * duration_s
    return int(math.ceil((mu + 8.0 * math.sqrt(mu) + 64.0) * scale))


def pack(specs: list, table: TableArrays, scale: float = 1.0, list_caps=None) -> PackedBatch:
    """specs: list of scenario dicts. list_caps (optional): exact per-model
    list capacities (e.g. counts of caller-supplied arrivals)."""
    n_scen = len(specs)
    n_models = sum(len(s["deployed"]) for s in specs)
    scen = (_abi.Scenario * max(n_scen, 1))()
    mods = (_abi.Model * max(n_models, 1))()
    req_off = list_off = seg_off = 0
    g = 0
    names = []
    cap_max = 1
    max_req_cap = 0
    for si, spec in enumerate(specs):
        dep = spec["deployed"]
        ids = [d["model_id"] for d in dep]
        # duplicates only for internal drivers whose batches never tie on a
        # WINDOW heap key (full_overlap_ratios: every batch emits at max_bs)
        if len(set(ids)) != len(ids) and not spec.get("allow_duplicate_models"):
            raise ValueError("duplicate model_id in deployed list")
        names.append(ids)
        order = sorted(range(len(ids)), key=lambda i: ids[i])
        rank = {i: r for r, i in enumerate(order)}
        orc = spec.get("oracle", {})
        S = scen[si]
        S.n_models = len(ids)
        S.model_off = g
        S.max_bs = int(spec.get("max_batch_size", 8))
        S.cap = int(spec.get("concurrency_cap", 2))
        S.duration_s = float(spec["duration_s"])
        S.window_ms = float(spec.get("batching_window_ms", 2.0))
        S.sigma = float(orc.get("noise_sigma", 0.05))
        S.beta[0] = float(orc.get("beta_l2", 1.0))
        S.beta[1] = float(orc.get("beta_dram", 1.5))
        S.beta[2] = float(orc.get("beta_sm", 0.5))
        S.seed = int(spec.get("seed", 0))
        S.oracle_seed = int(orc.get("seed", 0))
        S.batch_id_base = int(spec.get("batch_id_base", 0))
        if S.max_bs > table.max_bs:
            raise ValueError(f"max_batch_size {S.max_bs} exceeds the profile table's {table.max_bs}")
        req_cap = 0
        for mi, d in enumerate(dep):
            M = mods[g]
            if d["model_id"] not in table.models:
                raise ValueError(f"deployed models not in profile table: {[d['model_id']]}")
            M.entry_base = table.models.index(d["model_id"]) * table.max_bs
            M.name_rank = rank[mi]
            M.crc = zlib.crc32(d["model_id"].encode("utf-8"))
            M.rate_rps = float(d["arrival_rate_rps"])
            M.slo_ms = float(d["slo_ms"])
            M.scen = si
            M.list_off = list_off
            lc = list_caps[g] if list_caps is not None else _list_capacity(M.rate_rps, S.duration_s, scale)
            M.list_cap = int(lc)
            list_off += M.list_cap + (M.list_cap & 1)  # even offsets: 16-byte aligned list rows
            req_cap += M.list_cap
            g += 1
        S.req_off, S.req_cap = req_off, req_cap
        S.seg_off, S.seg_cap = seg_off, req_cap * (2 * S.cap - 1)
        req_off += req_cap
        seg_off += S.seg_cap
        cap_max = max(cap_max, S.cap)
        max_req_cap = max(max_req_cap, req_cap)
    return PackedBatch(specs=list(specs), table=table, scen=scen, models=mods, names=names, n_scen=n_scen,
                       n_models=n_models, total_req=req_off, total_list=list_off, total_seg=seg_off,
                       max_req_cap=max_req_cap, cap_max=cap_max)


# (field, dtype, size key) of every replay buffer; size keys resolved by sizes()
BUFFER_PLAN = [
    ("arr_t", np.float64, "req"), ("arr_model", np.int32, "req"),
    ("list_t", np.float64, "list"), ("list_rid", np.int32, "list"),
    ("n_req", np.int32, "scen"), ("n_list", np.int32, "models"),
    ("b_model", np.int32, "req"), ("b_size", np.int32, "req"), ("b_formed", np.float64, "req"),
    ("b_start", np.float64, "req"), ("b_completion", np.float64, "req"), ("b_measured", np.float64, "req"),
    ("b_seg_off", np.int32, "req"), ("b_nseg", np.int32, "req"), ("out_order", np.int32, "req"),
    ("b_running", np.int32, "req"),
    ("r_batch", np.int32, "req"), ("r_slo_met", np.uint8, "req"),
    ("s_tbegin", np.float64, "seg"), ("s_tend", np.float64, "seg"), ("s_slowdown", np.float64, "seg"),
    ("s_colo", np.float64, "seg3"),
    ("n_batches", np.int32, "scen"), ("n_segments", np.int32, "scen"), ("n_reseats", np.int32, "scen"),
    ("status", np.int32, "scen"), ("slot_seg", np.float64, "slots"), ("noise_tab", np.float64, "noise"),
    ("mb_t", np.float64, "list"), ("mb_info", np.int32, "list4"), ("n_mb", np.int32, "models"),
    ("slo_ws", np.int32, "slows"), ("form_ws", np.int32, "list3"), ("order", np.int32, "scen1"),
]


def sizes(pb: PackedBatch, seg_stride: int, noise_k: int = 0) -> dict:
    return {
        "noise": max(pb.total_req, 1) * max(noise_k, 1),
        "req": max(pb.total_req, 1), "list": max(pb.total_list, 1), "list4": 4 * max(pb.total_list, 1),
        "list3": 3 * max(pb.total_list, 1),
        "scen": max(pb.n_scen, 1), "scen1": pb.n_scen + 1,
        "models": max(pb.n_models, 1), "seg": max(pb.total_seg, 1), "seg3": 3 * max(pb.total_seg, 1),
        "slots": max(pb.n_scen, 1) * pb.cap_max * seg_stride * 5,
        "slows": _abi.SLO_WS_INTS,
    }
