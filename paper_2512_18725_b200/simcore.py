"""Scheduler replay.  Mirrors `intfsim.simcore` (`simcore.py:22-369`).

`run_scenario` / `run_scenarios` replay on the GPU: per-model batch
formation, FIFO capped admission, piecewise-constant interference segments
with bit-exact noise, SLO records (one warp per scenario, or busy-period jobs
for long traces; the reference's heap is replaced by an exact heap-free
recurrence, see csrc/replay_core.cuh and csrc/replay_warp.cuh).  Results are materialised as the reference's objects;
`ScenarioResult.arrays` keeps the flat arrays for batched reuse.

`GpuState` is the reference's interactive step API (`simcore.py:103-208`):
a host state machine (running list, completion heap, generations) whose
arithmetic -- the noise draw and the slowdown -- runs on the device through
the same entry points as the replay (`intf_noise_draws`, `intf_slowdowns`),
so a hand-driven GpuState reproduces the replay's segments bit for bit.
`run_scenario` always replays on the device; when a caller has instrumented
the step API (e.g. the reference's spy tests wrap `GpuState.dispatch`), it
additionally drives a GpuState along the device's own formation trace so the
hooks observe every dispatch and completion, and checks that walk against
the device replay bit for bit (`_drive_step_api`).
"""
from __future__ import annotations

import heapq
import itertools
from collections import deque
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
class RunningBatch:
    """A dispatched batch on the simulated GPU (`simcore.py:34-69`)."""

    batch: object  # batcher.BatchRequest
    profile: object  # profiles.ModelProfile
    start_time_ms: float
    total_work_ms: float
    progress_ms: float = 0.0
    segments: list = field(default_factory=list)
    completion_gen: int = 0

    @property
    def batch_id(self) -> int:
        return self.batch.batch_id

    @property
    def remaining_work_ms(self) -> float:
        return self.total_work_ms - self.progress_ms

    @property
    def current_slowdown(self) -> float:
        return self.segments[-1].slowdown

    def close_segment(self, now_ms: float) -> None:
        """End the open segment at now; a zero-length one is dropped, so the
        next reseat reuses its noise index (`simcore.py:56-66`)."""
        seg = self.segments[-1]
        if seg.t_end is not None:
            raise SimulationError(f"batch {self.batch_id}: segment already closed")
        if now_ms == seg.t_begin:
            self.segments.pop()
            return
        seg.t_end = now_ms
        self.progress_ms += (seg.t_end - seg.t_begin) / seg.slowdown

    def open_segment(self, now_ms: float, slowdown: float, colo) -> None:
        self.segments.append(Segment(t_begin=now_ms, t_end=None, slowdown=slowdown, colo=colo))


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


# event kinds in tie-break order at equal times (`simcore.py:98-100`)
_COMPLETION, _WINDOW, _ARRIVAL = 0, 1, 2


def _queue_key(model_id: str) -> int:
    """WINDOW heap key: crc32 of the model id (`simcore.py:313-316`)."""
    from .profiles import _stable_id

    return _stable_id(model_id)


class GpuState:
    """Simulated GPU for hand-driven stepping (`simcore.py:103-208`): a
    running list under the concurrency cap and a completion heap keyed
    (time, kind, key, push order).  Colo sums are added in running-list order
    from zeros on the host (plain fp64 adds, as numpy does); the noise draw
    and the slowdown are evaluated on the device."""

    def __init__(self, concurrency_cap: int, oracle):
        self.now_ms = 0.0
        self.concurrency_cap = concurrency_cap
        self.oracle = oracle
        self.running: list = []
        self.events: list = []
        self.outcomes: list = []
        self._push_seq = itertools.count()

    def push_event(self, time_ms: float, kind: int, key: int, payload) -> None:
        if time_ms < self.now_ms - 1e-9:
            raise SimulationError(f"event at {time_ms} scheduled in the past (now={self.now_ms})")
        heapq.heappush(self.events, (time_ms, kind, key, next(self._push_seq), payload))

    def colo_sums_for(self, rb: RunningBatch) -> np.ndarray:
        total = np.zeros(3)
        for other in self.running:
            if other is not rb:
                total += other.profile.throughputs()
        return total

    def _reseat(self, rb: RunningBatch) -> None:
        """New segment from now at the current co-location; reschedule the
        completion (`simcore.py:133-141`)."""
        from .interference import oracle_slowdown

        colo = self.colo_sums_for(rb)
        noise = self.oracle.noise_draw(rb.batch_id, len(rb.segments))
        slowdown = oracle_slowdown(rb.profile.throughputs(), colo, self.oracle, noise)
        rb.open_segment(self.now_ms, slowdown, colo)
        rb.completion_gen += 1
        self.push_event(self.now_ms + rb.remaining_work_ms * slowdown, _COMPLETION, rb.batch_id,
                        (rb, rb.completion_gen))

    def _colo_changed(self, survivors: list) -> None:
        for rb in survivors:
            rb.close_segment(self.now_ms)
            self._reseat(rb)

    def can_dispatch(self) -> bool:
        return len(self.running) < self.concurrency_cap

    def dispatch(self, batch, table) -> RunningBatch:
        """Start `batch` now: it is reseated first, then every survivor in
        running-list order (`simcore.py:150-171`)."""
        if not self.can_dispatch():
            raise SimulationError(f"dispatch of batch {batch.batch_id} at concurrency cap {self.concurrency_cap}")
        profile = table.get(batch.model_id, batch.batch_size)
        rb = RunningBatch(batch=batch, profile=profile, start_time_ms=self.now_ms,
                          total_work_ms=profile.solo_duration_ms)
        survivors = list(self.running)
        self.running.append(rb)
        self._reseat(rb)
        self._colo_changed(survivors)
        return rb

    def complete(self, rb: RunningBatch) -> BatchOutcome:
        """Finish rb now and reseat the survivors (`simcore.py:173-198`)."""
        rb.close_segment(self.now_ms)
        if abs(rb.progress_ms - rb.total_work_ms) > 1e-6 * rb.total_work_ms:
            raise SimulationError(f"batch {rb.batch_id} completed with progress {rb.progress_ms} "
                                  f"!= work {rb.total_work_ms}")
        self.running.remove(rb)
        measured = self.now_ms - rb.start_time_ms
        if all(seg.slowdown == 1.0 for seg in rb.segments):
            measured = rb.total_work_ms  # unit slowdown throughout: measured == profiled by identity
        out = BatchOutcome(rb.batch_id, rb.batch.model_id, rb.batch.batch_size, rb.start_time_ms, measured,
                           rb.total_work_ms, self.now_ms, rb.segments)
        self.outcomes.append(out)
        self._colo_changed(list(self.running))
        return out

    def advance_to_next_event(self):
        """Pop the earliest event; now = max(now, its time) (`simcore.py:200-208`)."""
        if not self.events:
            raise SimulationError("advance with an empty event queue")
        time_ms, kind, key, _, payload = heapq.heappop(self.events)
        if time_ms < self.now_ms - 1e-9:
            raise SimulationError(f"event at {time_ms} is in the past ({self.now_ms})")
        self.now_ms = max(self.now_ms, time_ms)
        return time_ms, kind, key, payload


_STEP_API = {n: GpuState.__dict__[n] for n in ("push_event", "colo_sums_for", "_reseat", "_colo_changed",
                                                 "can_dispatch", "dispatch", "complete", "advance_to_next_event")}


def _step_api_instrumented() -> bool:
    return any(GpuState.__dict__.get(n) is not f for n, f in _STEP_API.items())


def _drive_step_api(spec, table, v) -> list:
    """Drive a GpuState through one scenario along the device replay's
    formation trace (batch ids, members and formation times from
    `intf_form_batches`): formations and completions merged by (time, kind),
    FIFO dispatch after every event (`simcore.py:258-300`).  Instrumented
    step-API methods therefore see every dispatch and completion.  Returns
    the outcomes in (completion, batch_id) order."""
    from .batcher import BatchRequest
    from .workload import RequestEvent

    ids = [d.model_id for d in spec.deployed]
    slo = [d.slo_ms for d in spec.deployed]
    at, am, rb_of = v["arr_t"], v["arr_model"], v["r_batch"]
    members = [[] for _ in range(len(v["b_model"]))]
    for r in range(len(at)):
        m = int(am[r])
        members[int(rb_of[r])].append(RequestEvent(r, ids[m], float(at[r]), float(at[r]) + slo[m]))
    batches = [BatchRequest(b, ids[int(v["b_model"][b])], tuple(members[b]), float(v["b_formed"][b]))
               for b in range(len(members))]
    state = GpuState(spec.concurrency_cap, spec.oracle)
    queue = deque()
    i = 0
    while i < len(batches) or state.events:
        if state.events and (i == len(batches) or state.events[0][0] <= batches[i].formed_at_ms):
            _, _, _, (rb, gen) = state.advance_to_next_event()  # completions first at equal times
            if gen != rb.completion_gen or rb not in state.running:
                continue  # superseded by a later re-projection
            state.complete(rb)
        else:
            state.now_ms = max(state.now_ms, batches[i].formed_at_ms)
            queue.append(batches[i])
            i += 1
        while queue and state.can_dispatch():
            state.dispatch(queue.popleft(), table)
    state.outcomes.sort(key=lambda o: (o.completion_time_ms, o.batch_id))
    return state.outcomes


def _check_step_walk(name, walked, device) -> None:
    """The step-API walk must equal the device replay bit for bit."""
    same = len(walked) == len(device) and all(
        (a.batch_id, a.start_ms, a.measured_duration_ms, a.completion_time_ms, len(a.segments))
        == (b.batch_id, b.start_ms, b.measured_duration_ms, b.completion_time_ms, len(b.segments))
        and all((x.t_begin, x.t_end, x.slowdown) == (y.t_begin, y.t_end, y.slowdown)
                and np.array_equal(x.colo, y.colo) for x, y in zip(a.segments, b.segments))
        for a, b in zip(walked, device))
    if not same:
        raise SimulationError(f"scenario {name!r}: the step-API walk differs from the device replay")


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
    ta = table.arrays()
    pipe, h = engine.run_batch([scenario_to_dict(s) for s in specs], ta, preds=preds, arrivals=arrivals)
    for s, spec in enumerate(specs):
        if ta.missing:
            _check_rows(spec, ta, pipe.scenario(h, s))
        _raise_status(spec.name, int(h["status"][s]))
    return pipe, h


def _check_rows(spec, ta, v) -> None:
    """A dispatched batch whose (model, batch size) has no profile entry is
    the reference's ProfileError from `table.get` at dispatch
    (`simcore.py:155`, `profiles.py:60-64`); the first such batch in
    dispatch (= batch id) order is reported."""
    from .profiles import ProfileError

    ids = [d.model_id for d in spec.deployed]
    base = np.array([ta.models.index(m) * ta.max_bs for m in ids], dtype=np.int64)
    rows = base[v["b_model"]] + v["b_size"].astype(np.int64) - 1
    bad = np.flatnonzero(np.isin(rows, np.fromiter(ta.missing, dtype=np.int64)))
    if len(bad):
        b = int(bad[0])
        raise ProfileError(f"no profile for model {ids[v['b_model'][b]]!r} at batch size {int(v['b_size'][b])}")


def _materialize(spec, table, v) -> ScenarioResult:
    """The reference's result objects from the flat device arrays: outcomes in
    (completion, batch_id) order with their segments, records by request id,
    samples in outcome order.  Vectorised gathers first, then one pass of
    object construction from Python lists (the per-object cost is the
    dataclass __init__ alone)."""
    ta = table.arrays()
    ids = [d.model_id for d in spec.deployed]
    order = np.asarray(v["order"], dtype=np.int64)
    bm, bsz = np.asarray(v["b_model"]), np.asarray(v["b_size"])
    base = np.array([ta.models.index(m) * ta.max_bs for m in ids], dtype=np.int64)
    rows = base[bm[order]] + bsz[order].astype(np.int64) - 1 if len(order) else np.zeros(0, np.int64)
    soff, nseg = v["b_seg_off"][order].astype(np.int64), v["b_nseg"][order].astype(np.int64)
    # segment records of every outcome, in outcome order (one gather)
    seg_start = np.concatenate([[0], np.cumsum(nseg)[:-1]]) if len(order) else np.zeros(0, np.int64)
    idx = (np.repeat(soff - seg_start, nseg) + np.arange(int(nseg.sum()))) if len(order) else np.zeros(0, np.int64)
    colo = np.array(v["s_colo"][idx], dtype=float).reshape(-1, 3)  # private copy; each Segment views its row
    tb, te, sd = v["s_tbegin"][idx].tolist(), v["s_tend"][idx].tolist(), v["s_slowdown"][idx].tolist()
    start, comp, meas = v["b_start"], v["b_completion"], v["b_measured"]
    o_start, o_comp, o_meas = start[order].tolist(), comp[order].tolist(), meas[order].tolist()
    o_prof, o_model, o_size = ta.solo[rows].tolist(), bm[order].tolist(), bsz[order].tolist()
    outcomes = OutcomeList()
    q = 0
    for k, b in enumerate(order.tolist()):
        n = int(nseg[k])
        segs = [Segment(tb[j], te[j], sd[j], colo[j]) for j in range(q, q + n)]
        q += n
        outcomes.append(BatchOutcome(b, ids[o_model[k]], o_size[k], o_start[k], o_meas[k], o_prof[k], o_comp[k], segs))
    outcomes.arrays = {
        "own": ta.thr[rows].reshape(-1, 3), "seg_off": seg_start.astype(np.int64), "nseg": nseg.astype(np.int32),
        "colo": colo, "measured": meas[order], "profiled": ta.solo[rows], "batch_id": order,
    }
    at, am, rb, met = v["arr_t"], v["arr_model"], v["r_batch"], v["r_slo_met"]
    r_t, r_model, r_b = at.tolist(), np.asarray(am).tolist(), np.asarray(rb).tolist()
    r_start, r_comp, r_met = start[rb].tolist(), comp[rb].tolist(), np.asarray(met, dtype=bool).tolist()
    records = [RequestRecord(i, ids[r_model[i]], r_t[i], r_b[i], r_start[i], r_comp[i], r_met[i])
               for i in range(len(r_t))]
    samples = samples_from_outcomes(outcomes, table, spec.colocation_mode, scenario=spec.name)
    return ScenarioResult(outcomes=outcomes, records=records, samples=samples, arrays=dict(v))


def run_scenarios(specs, table) -> list:
    """Replay many scenarios in one batched device pass."""
    specs = list(specs)
    pipe, h = run_scenarios_arrays(specs, table)
    out = []
    for s, spec in enumerate(specs):
        v = pipe.scenario(h, s)
        res = _materialize(spec, table, v)
        if _step_api_instrumented():
            _check_step_walk(spec.name, _drive_step_api(spec, table, v), res.outcomes)
        out.append(res)
    return out


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
