"""Golden fixture access (tests/golden/*.npz, made by tests/golden/make_golden.py
from the unmodified reference)."""
from __future__ import annotations

import functools
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MODES = [(0, 1.0), (1, 1.0 / 3.0), (1, 0.5), (1, 2.0 / 3.0)]  # static, EWMA 1/3, 1/2, 2/3


@functools.lru_cache(maxsize=None)
def load(name: str):
    return np.load(os.path.join(HERE, name))


def replay():
    return load("replay_golden.npz")


def table(name: str = "default"):
    from paper_2512_18725_b200._pack import TableArrays

    G = replay()
    return TableArrays(list(G[f"_table/{name}/models"]), int(G[f"_table/{name}/max_bs"]), G[f"_table/{name}/solo"],
                       G[f"_table/{name}/thr"])


def table_names():
    G = replay()
    return sorted({str(G[n + "/table"]) for n in G["_names"]})


def scenario_names(table_name: str | None = None):
    G = replay()
    names = [str(n) for n in G["_names"]]
    if table_name is None:
        return names
    return [n for n in names if str(G[n + "/table"]) == table_name]


def spec(name: str) -> dict:
    return json.loads(str(replay()[name + "/spec"]))


def outcome_segment_index(seg_off, nseg, order):
    if len(order) == 0:
        return np.zeros(0, dtype=np.int64)
    return np.concatenate([np.arange(seg_off[b], seg_off[b] + nseg[b]) for b in order])


def compare_replay(v: dict, name: str) -> list:
    """Bit-exact comparison of a replay view (oracle.run_scenario key layout)
    with the golden outputs of scenario `name`; returns failing fields."""
    G = replay()
    p = name + "/"
    o = np.asarray(v["order"])
    idx = outcome_segment_index(v["b_seg_off"], v["b_nseg"], o)
    checks = {
        "arrivals": np.array_equal(v["arr_t"], G[p + "arr_t"]) and np.array_equal(v["arr_model"], G[p + "arr_model"]),
        "batch_order": np.array_equal(o, G[p + "o_batch"]),
        "model": np.array_equal(v["b_model"][o], G[p + "o_model"]),
        "size": np.array_equal(v["b_size"][o], G[p + "o_size"]),
        "start": np.array_equal(v["b_start"][o], G[p + "o_start"]),
        "measured": np.array_equal(v["b_measured"][o], G[p + "o_measured"]),
        "completion": np.array_equal(v["b_completion"][o], G[p + "o_completion"]),
        "n_segments": np.array_equal(v["b_nseg"][o], G[p + "o_nseg"]),
        "request_batch": np.array_equal(v["r_batch"], G[p + "r_batch"]),
        "seg_tbegin": np.array_equal(v["s_tbegin"][idx], G[p + "s_tbegin"]),
        "seg_tend": np.array_equal(v["s_tend"][idx], G[p + "s_tend"]),
        "seg_slowdown": np.array_equal(v["s_slowdown"][idx], G[p + "s_slowdown"]),
        "seg_colo": np.array_equal(v["s_colo"][idx], G[p + "s_colo"]),
    }
    if "r_slo_met" in v:
        checks["slo_met"] = np.array_equal(v["r_slo_met"], G[p + "r_slo"])
    return [k for k, ok in checks.items() if not ok]
