"""Byte-identical CSV artifacts of a replay.

The reference CLI's `simulate` (`cli.py:72-125`) writes, per scenario and
seed, arrivals / outcomes / requests / samples / slo_report (/ segments)
CSVs through `csv.writer` with Python `repr(float)` fields (row helpers
`workload.py:173-178`, `simcore.py:319-369`, `metrics.py:82-128`,
`colocation.py:108-126`).  Here the rows come straight from the device
replay's flat arrays (no per-row Python objects) and are formatted by the
native `intf_csv_rows` (csrc/csv.cu: shortest round-trip repr, csv.writer's
quoting and "\\r\\n" terminators), so a 10^6-request trace materialises in
well under a second and the files hash identically to the reference's.
"""
from __future__ import annotations

import ctypes
import hashlib
import json
from pathlib import Path

import numpy as np

from . import _abi

COL_I64, COL_F64, COL_STR, COL_NPF64 = 0, 1, 2, 3

ARRIVAL_CSV_HEADER = ["request_id", "model_id", "arrival_time_ms", "deadline_ms"]
OUTCOME_CSV_HEADER = ["batch_id", "model_id", "batch_size", "start_ms", "measured_ms", "profiled_ms",
                      "interference_ratio", "n_segments"]
SEGMENT_CSV_HEADER = ["batch_id", "segment_index", "t_begin_ms", "t_end_ms", "slowdown", "colo_l2", "colo_dram",
                      "colo_sm"]
REQUEST_CSV_HEADER = ["request_id", "model_id", "arrival_ms", "dispatch_ms", "completion_ms", "latency_ms",
                      "queueing_ms", "slo_met"]
REPORT_CSV_HEADER = ["model_id", "n_requests", "slo_satisfaction", "p50_latency_ms", "p95_latency_ms",
                     "p99_latency_ms"]
SAMPLE_CSV_HEADER = ["batch_id", "scenario", "own_l2", "own_dram", "own_sm", "colo_l2", "colo_dram", "colo_sm",
                     "y_ratio", "mode", "alpha"]
TOOL_VERSION = "0.1.0"  # the reference's intfsim.__version__ (`__init__.py:5`), recorded in manifest.json


def csv_quote(field: str) -> str:
    """csv.writer's QUOTE_MINIMAL for one string field (default dialect)."""
    if any(c in field for c in ',"\r\n'):
        return '"' + field.replace('"', '""') + '"'
    return field


def repr_f64(v: float) -> str:
    """CPython repr(float), computed by the native formatter."""
    buf = ctypes.create_string_buffer(40)
    _abi.check(_abi.load().intf_repr_f64(float(v), buf, 40), "intf_repr_f64")
    return buf.value.decode()


def format_rows(columns, header=None) -> bytes:
    """CSV bytes of typed columns: (COL_I64, int array) | (COL_F64, float
    array) | (COL_NPF64, float array) | (COL_STR, (int32 indices, strings))."""
    n = len(columns[0][1][0]) if columns[0][0] == COL_STR else len(columns[0][1])
    kinds = (ctypes.c_int32 * len(columns))()
    ptrs = (ctypes.c_void_p * len(columns))()
    keep, strings = [], []
    for c, (kind, data) in enumerate(columns):
        kinds[c] = kind
        if kind == COL_STR:
            idx, tab = data
            a = np.ascontiguousarray(np.asarray(idx, dtype=np.int32) + len(strings))
            strings.extend(csv_quote(str(x)) for x in tab)
        elif kind == COL_I64:
            a = np.ascontiguousarray(data, dtype=np.int64)
        else:
            a = np.ascontiguousarray(data, dtype=np.float64)
        if len(a) != n:
            raise ValueError("format_rows: columns differ in length")
        keep.append(a)
        ptrs[c] = a.ctypes.data
    enc = [s.encode() for s in strings]
    stab = (ctypes.c_char_p * max(len(enc), 1))(*enc)
    slen = (ctypes.c_int32 * max(len(enc), 1))(*[len(e) for e in enc])
    L = _abi.load()
    need = ctypes.c_int64(0)
    _abi.check(L.intf_csv_rows(n, len(columns), kinds, ptrs, stab, slen, None, 0, ctypes.byref(need)),
               "intf_csv_rows")
    buf = ctypes.create_string_buffer(max(int(need.value), 1))
    _abi.check(L.intf_csv_rows(n, len(columns), kinds, ptrs, stab, slen, buf, need.value, ctypes.byref(need)),
               "intf_csv_rows")
    body = buf.raw[: need.value]
    if header is not None:
        body = (",".join(csv_quote(h) for h in header) + "\r\n").encode() + body
    return body


# ------------------------------------------------------------------ files
def _arrays(table):
    """ProfileTable or its packed TableArrays."""
    return table.arrays() if hasattr(table, "arrays") else table


def _ids(spec):
    return [d.model_id for d in spec.deployed]


def arrivals_csv(spec, v) -> bytes:
    """`workload.py:173-178`: deadline = arrival + slo (`workload.py:103`)."""
    am = np.asarray(v["arr_model"], dtype=np.int64)
    at = np.asarray(v["arr_t"], dtype=np.float64)
    slo = np.array([d.slo_ms for d in spec.deployed], dtype=np.float64)
    return format_rows([(COL_I64, np.arange(len(at))), (COL_STR, (am, _ids(spec))), (COL_F64, at),
                        (COL_F64, at + slo[am])], ARRIVAL_CSV_HEADER)


def _outcome_rows(spec, table, v):
    ta = _arrays(table)
    ids = _ids(spec)
    order = np.asarray(v["order"], dtype=np.int64)
    bm = np.asarray(v["b_model"])[order]
    bsz = np.asarray(v["b_size"])[order]
    rows = np.array([ta.row(ids[m], int(b)) for m, b in zip(bm, bsz)], dtype=np.int64)
    prof = np.asarray(ta.solo, dtype=np.float64)[rows] if len(rows) else np.zeros(0)
    return order, bm, bsz, prof


def outcomes_csv(spec, table, v) -> bytes:
    """`simcore.py:319-340`; interference_ratio = measured / profiled (`simcore.py:80-82`)."""
    order, bm, bsz, prof = _outcome_rows(spec, table, v)
    meas = np.asarray(v["b_measured"])[order]
    return format_rows([(COL_I64, order), (COL_STR, (bm, _ids(spec))), (COL_I64, bsz),
                        (COL_F64, np.asarray(v["b_start"])[order]), (COL_F64, meas), (COL_F64, prof),
                        (COL_F64, meas / prof), (COL_I64, np.asarray(v["b_nseg"])[order])], OUTCOME_CSV_HEADER)


def _segment_index(v):
    order = np.asarray(v["order"], dtype=np.int64)
    off = np.asarray(v["b_seg_off"], dtype=np.int64)[order]
    ns = np.asarray(v["b_nseg"], dtype=np.int64)[order]
    if ns.sum() == 0:
        return order, ns, np.zeros(0, np.int64), np.zeros(0, np.int64)
    start = np.repeat(np.cumsum(ns) - ns, ns)
    within = np.arange(int(ns.sum())) - start
    return order, ns, np.repeat(off, ns) + within, within


def segments_csv(spec, v) -> bytes:
    """`simcore.py:343-369`: one row per kept segment, outcome order."""
    order, ns, idx, within = _segment_index(v)
    colo = np.asarray(v["s_colo"]).reshape(-1, 3)[idx]
    return format_rows([(COL_I64, np.repeat(order, ns)), (COL_I64, within),
                        (COL_F64, np.asarray(v["s_tbegin"])[idx]), (COL_F64, np.asarray(v["s_tend"])[idx]),
                        (COL_F64, np.asarray(v["s_slowdown"])[idx]), (COL_F64, colo[:, 0]), (COL_F64, colo[:, 1]),
                        (COL_F64, colo[:, 2])], SEGMENT_CSV_HEADER)


def requests_csv(spec, v) -> bytes:
    """`metrics.py:82-106`: latency = completion - arrival, queueing =
    dispatch - arrival (`metrics.py:19-25`), records by request id."""
    at = np.asarray(v["arr_t"], dtype=np.float64)
    rb = np.asarray(v["r_batch"], dtype=np.int64)
    disp = np.asarray(v["b_start"])[rb]
    comp = np.asarray(v["b_completion"])[rb]
    return format_rows([(COL_I64, np.arange(len(at))), (COL_STR, (np.asarray(v["arr_model"]), _ids(spec))),
                        (COL_F64, at), (COL_F64, disp), (COL_F64, comp), (COL_F64, comp - at),
                        (COL_F64, disp - at), (COL_I64, np.asarray(v["r_slo_met"], dtype=np.int64))],
                       REQUEST_CSV_HEADER)


def slo_report_csv(spec, v, report=None) -> bytes:
    """`metrics.py:109-128` over the device SLO report (`metrics.py:49-79`).
    report: optional precomputed rows [(model, n, satisfaction, p50, p95, p99)]."""
    if report is None:
        from .metrics import slo_report_arrays

        dep = _ids(spec)
        ids = sorted(set(dep[m] for m in np.asarray(v["arr_model"])))
        pos = {m: i for i, m in enumerate(ids)}
        group = np.array([pos[dep[m]] for m in np.asarray(v["arr_model"])], dtype=np.int32)
        rb = np.asarray(v["r_batch"], dtype=np.int64)
        rep = slo_report_arrays(ids, group, v["arr_t"], np.asarray(v["b_completion"])[rb], v["r_slo_met"])
        report = [(m, r.n_requests, r.slo_satisfaction, r.p50_latency_ms, r.p95_latency_ms, r.p99_latency_ms)
                  for m, r in rep.items()]
    r = sorted(report)
    return format_rows([(COL_STR, (np.arange(len(r)), [x[0] for x in r]))] +
                       [(COL_I64 if j == 1 else COL_F64, [x[j] for x in r]) for j in range(1, 6)],
                       REPORT_CSV_HEADER)


def samples_csv(spec, table, v, features=None) -> bytes:
    """`colocation.py:108-126`: features of the scenario's co-location mode,
    computed on the device (`colocation.py:95-105`) unless `features` = (X,
    y) in outcome order is given; the reference formats the feature entries
    with "%r" of numpy scalars."""
    from . import engine
    from .colocation import EWMA

    mode = spec.colocation_mode
    order, bm, bsz, prof = _outcome_rows(spec, table, v)
    _, ns, idx, _ = _segment_index(v)
    ta = _arrays(table)
    ids = _ids(spec)
    rows = np.array([ta.row(ids[m], int(b)) for m, b in zip(bm, bsz)], dtype=np.int64)
    own = np.asarray(ta.thr, dtype=np.float64).reshape(-1, 3)[rows] if len(rows) else np.zeros((0, 3))
    colo = np.asarray(v["s_colo"]).reshape(-1, 3)[idx]
    meas = np.asarray(v["b_measured"])[order]
    n = len(order)
    if features is not None:
        X, y = (np.asarray(a, dtype=np.float64) for a in features)
        X = X.reshape(n, 6)
    elif n:
        seg_off = (np.cumsum(ns) - ns).astype(np.int64)
        X, y, _ = engine.features_rows(own, seg_off, ns.astype(np.int32), colo, meas, prof, [mode.predictor()])
        X = X[0]
    else:
        X, y = np.zeros((0, 6)), np.zeros(0)
    kinds = [mode.kind]
    alpha = [repr(float(mode.alpha)) if mode.kind == EWMA else ""]
    cols = [(COL_I64, order), (COL_STR, (np.zeros(n, np.int32), [spec.name]))]
    cols += [(COL_NPF64, X[:, j]) for j in range(6)]
    cols += [(COL_F64, y), (COL_STR, (np.zeros(n, np.int32), kinds)), (COL_STR, (np.zeros(n, np.int32), alpha))]
    return format_rows(cols, SAMPLE_CSV_HEADER)


def scenario_csvs(spec, table, v, segments: bool = False, features=None, report=None) -> dict:
    """{file name: bytes} for one replayed scenario, as `cmd_simulate` writes
    them (`cli.py:85-122`); v = the replay's flat arrays (engine
    ReplayPipeline.scenario layout)."""
    out = {"arrivals.csv": arrivals_csv(spec, v), "outcomes.csv": outcomes_csv(spec, table, v),
           "requests.csv": requests_csv(spec, v), "samples.csv": samples_csv(spec, table, v, features)}
    if len(np.asarray(v["arr_t"])):
        out["slo_report.csv"] = slo_report_csv(spec, v, report)
    if segments:
        out["segments.csv"] = segments_csv(spec, v)
    return out


def simulate(profiles, scenarios, out, seeds=(0,), segments: bool = False, verbose: bool = True) -> dict:
    """The reference's `intfsim simulate` (`cli.py:72-125`) through the
    device replay: every (scenario, seed) pair is replayed in ONE batched
    launch sequence, then materialised.  Returns {run dir: {file: sha256}}."""
    from dataclasses import replace

    from .profiles import load_profiles
    from .simcore import run_scenarios_arrays
    from .workload import load_scenario

    table = load_profiles(profiles)
    out_root = Path(out)
    config = {"profiles": str(profiles), "scenarios": [str(s) for s in scenarios], "seeds": list(seeds),
              "segments": segments}
    blob = json.dumps(config, sort_keys=True).encode("utf-8")
    out_root.mkdir(parents=True, exist_ok=True)
    (out_root / "manifest.json").write_text(json.dumps({"config_sha256": hashlib.sha256(blob).hexdigest(),
                                                        "seeds": list(seeds), "tool_version": TOOL_VERSION},
                                                       indent=2) + "\n", encoding="utf-8")
    runs = [replace(load_scenario(p, table), seed=s) for p in scenarios for s in seeds]
    pipe, h = run_scenarios_arrays(runs, table)
    hashes = {}
    for i, spec in enumerate(runs):
        v = pipe.scenario(h, i)
        d = out_root / f"{spec.name}_seed{spec.seed}"
        d.mkdir(parents=True, exist_ok=True)
        files = scenario_csvs(spec, table, v, segments)
        for name, data in files.items():
            (d / name).write_bytes(data)
        hashes[str(d)] = {k: hashlib.sha256(b).hexdigest() for k, b in files.items()}
        if verbose:
            print(f"{spec.name} seed={spec.seed}: {len(np.asarray(v['arr_t']))} requests, "
                  f"{len(np.asarray(v['order']))} batches -> {d}")
    return hashes


def sha256_dir(d) -> dict:
    return {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted(Path(d).glob("*.csv"))}
