"""Scheduler replay.  Mirrors `intfsim.simcore` (`simcore.py:22-369`).

`run_scenario` / `run_scenarios` replay on the GPU: per-model batch
formation, FIFO capped admission, piecewise-constant interference segments
with bit-exact noise, SLO records (one CUDA thread per scenario; the
reference's heap is replaced by an exact heap-free recurrence, see
csrc/replay_core.cuh).  Results are materialised as the reference's objects;
`ScenarioResult.arrays` keeps the flat arrays for batched reuse.

`GpuState` (the reference's interactive step API, `simcore.py:103-208`) is
not provided: its semantics are the replay kernel's, reached through
`run_scenario` (out of scope).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .colocation import samples_from_outcomes
from .metrics import RequestRecord


class SimulationError(RuntimeError):
    """Invariant violation in the replay (`simcore.py:22`)."""


@dataclass
class Segment:
    t_begin: float
    t_end: float | None
    slowdown: float
    colo: np.ndarray


@dataclass
class BatchOutcome:
    batch_id: int
    model_id: str
    batch_size: int
    start_ms: float
    measured_duration_ms: float
    profiled_ms: float
    completion_time_ms: float
    segments: list

    @property
    def interference_ratio(self) -> float:
        return self.measured_duration_ms / self.profiled_ms

    @property
    def colo_history(self) -> list:
        return [s.colo for s in self.segments]

    @property
    def n_segments(self) -> int:
        return len(self.segments)


class OutcomeList(list):
    """Outcomes in (completion, batch_id) order plus their flat arrays
    (`own`, `seg_off`, `nseg`, `colo`, `measured`, `profiled`, `batch_id`)."""

    arrays: dict | None = None


@dataclass
class ScenarioResult:
    outcomes: list
    records: list
    samples: list
    arrays: dict = field(default_factory=dict, repr=False)


_STATUS_TEXT = [(1, "event scheduled in the past"), (2, "dispatch at concurrency cap / unsupported scenario shape"),
                (4, "batch completed with progress != work"),
                (8, "simulation drained its event queue before quiescence")]


def _raise_status(name: str, st: int) -> None:
    msgs = [m for bit, m in _STATUS_TEXT if st & bit]
    if msgs:
        raise SimulationError(f"scenario {name!r}: " + "; ".join(msgs))


def _check_models(spec, table):
    missing = [d.model_id for d in spec.deployed if d.model_id not in table.models()]
    if missing:
        raise SimulationError(f"deployed models not in profile table: {missing}")


def run_scenarios_arrays(specs, table, preds=(), arrivals=None):
    """Batched replay -> (pipeline, fetched host buffers).  One launch per
    pipeline stage for all scenarios."""
    from . import engine
    from .workload import scenario_to_dict

    for s in specs:
        _check_models(s, table)
    pipe, h = engine.run_batch([scenario_to_dict(s) for s in specs], table.arrays(), preds=preds, arrivals=arrivals)
    for s, spec in enumerate(specs):
        _raise_status(spec.name, int(h["status"][s]))
    return pipe, h


def _materialize(spec, table, v) -> ScenarioResult:
    ta = table.arrays()
    dep = spec.deployed
    ids = [d.model_id for d in dep]
    order = np.asarray(v["order"])
    bm, bsz = v["b_model"], v["b_size"]
    rows = np.array([ta.row(ids[bm[b]], int(bsz[b])) for b in order], dtype=np.int64)
    soff, nseg = v["b_seg_off"][order].astype(np.int64), v["b_nseg"][order].astype(np.int32)
    colo = v["s_colo"]
    outcomes = OutcomeList()
    tb, te, sd = v["s_tbegin"], v["s_tend"], v["s_slowdown"]
    start, comp, meas = v["b_start"], v["b_completion"], v["b_measured"]
    for k, b in enumerate(order.tolist()):
        o, n = int(soff[k]), int(nseg[k])
        segs = [Segment(float(tb[q]), float(te[q]), float(sd[q]), colo[q].copy()) for q in range(o, o + n)]
        outcomes.append(BatchOutcome(b, ids[bm[b]], int(bsz[b]), float(start[b]), float(meas[b]),
                                     float(ta.solo[rows[k]]), float(comp[b]), segs))
    # compact colo histories in outcome order for batched feature reuse
    idx = np.concatenate([np.arange(o, o + n) for o, n in zip(soff, nseg)]) if len(order) else np.zeros(0, np.int64)
    outcomes.arrays = {
        "own": ta.thr[rows].reshape(-1, 3), "seg_off": np.concatenate([[0], np.cumsum(nseg)[:-1]]).astype(np.int64)
        if len(order) else np.zeros(0, np.int64), "nseg": nseg, "colo": colo[idx].reshape(-1, 3),
        "measured": meas[order], "profiled": ta.solo[rows], "batch_id": order.astype(np.int64),
    }
    at, am, rb, met = v["arr_t"], v["arr_model"], v["r_batch"], v["r_slo_met"]
    records = [RequestRecord(i, ids[am[i]], float(at[i]), int(rb[i]), float(start[rb[i]]), float(comp[rb[i]]),
                             bool(met[i])) for i in range(len(at))]
    samples = samples_from_outcomes(outcomes, table, spec.colocation_mode, scenario=spec.name)
    return ScenarioResult(outcomes=outcomes, records=records, samples=samples, arrays=dict(v))


def run_scenarios(specs, table) -> list:
    """Replay many scenarios in one batched device pass."""
    specs = list(specs)
    pipe, h = run_scenarios_arrays(specs, table)
    return [_materialize(spec, table, pipe.scenario(h, s)) for s, spec in enumerate(specs)]


def run_scenario(spec, table) -> ScenarioResult:
    """arrivals -> batcher -> FIFO dispatch -> GPU to quiescence (`simcore.py:218-310`)."""
    return run_scenarios([spec], table)[0]


OUTCOME_CSV_HEADER = ["batch_id", "model_id", "batch_size", "start_ms", "measured_ms", "profiled_ms",
                      "interference_ratio", "n_segments"]


def outcome_csv_rows(outcomes):
    for o in outcomes:
        yield [o.batch_id, o.model_id, o.batch_size, repr(o.start_ms), repr(o.measured_duration_ms),
               repr(o.profiled_ms), repr(o.interference_ratio), o.n_segments]


SEGMENT_CSV_HEADER = ["batch_id", "segment_index", "t_begin_ms", "t_end_ms", "slowdown", "colo_l2", "colo_dram",
                      "colo_sm"]


def segment_csv_rows(outcomes):
    for o in outcomes:
        for i, s in enumerate(o.segments):
            yield [o.batch_id, i, repr(s.t_begin), repr(s.t_end), repr(s.slowdown), repr(float(s.colo[0])),
                   repr(float(s.colo[1])), repr(float(s.colo[2]))]
