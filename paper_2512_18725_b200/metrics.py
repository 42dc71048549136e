"""Per-request latency accounting and SLO reports.  Mirrors
`intfsim.metrics` (`metrics.py:9-128`); selection runs on the GPU (exact
nearest-rank via radix select on IEEE bit order)."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RequestRecord:
    request_id: int
    model_id: str
    arrival_ms: float
    batch_id: int
    dispatch_ms: float
    completion_ms: float
    slo_met: bool

    @property
    def latency_ms(self) -> float:
        return self.completion_ms - self.arrival_ms

    @property
    def queueing_ms(self) -> float:
        return self.dispatch_ms - self.arrival_ms


def percentile(values, p: float) -> float:
    """Nearest-rank percentile: the ceil(p/100 * n)-th smallest (`metrics.py:28-36`)."""
    from . import engine

    v = np.asarray(list(values) if not isinstance(values, np.ndarray) else values, dtype=float).reshape(-1)
    if v.size == 0:
        raise ValueError("percentile of empty list")
    if not (0.0 <= p <= 100.0):
        raise ValueError(f"percentile p={p} outside [0, 100]")
    return float(engine.quantiles(v, [float(p)])[0])


@dataclass(frozen=True)
class ModelLatencyReport:
    model_id: str
    n_requests: int
    slo_satisfaction: float
    p50_latency_ms: float
    p95_latency_ms: float
    p99_latency_ms: float


def slo_report_arrays(model_ids, group, arrival, completion, met, warmup_fraction: float = 0.0) -> dict:
    """slo_report over record arrays: group[i] indexes model_ids."""
    from . import engine

    arrival = np.asarray(arrival, dtype=float)
    if arrival.size == 0:
        raise ValueError("slo_report on empty record list")
    cutoff = -math.inf
    if warmup_fraction:
        t0, t1 = float(arrival.min()), float(arrival.max())
        cutoff = t0 + warmup_fraction * (t1 - t0)  # `metrics.py:62-65`
        if not np.any(arrival >= cutoff):
            cutoff = -math.inf  # `trimmed or records`
    n, m, p = engine.latency_report(group, arrival, completion, met, len(model_ids), cutoff)
    out = {}
    for g in sorted(range(len(model_ids)), key=lambda i: model_ids[i]):
        if n[g]:
            out[model_ids[g]] = ModelLatencyReport(model_ids[g], int(n[g]), int(m[g]) / int(n[g]), float(p[g, 0]),
                                                   float(p[g, 1]), float(p[g, 2]))
    return out


def slo_report(records, warmup_fraction: float = 0.0) -> dict:
    """Per-model SLO satisfaction and p50/p95/p99 latency (`metrics.py:49-79`)."""
    records = list(records)
    if not records:
        raise ValueError("slo_report on empty record list")
    ids = sorted({r.model_id for r in records})
    idx = {m: i for i, m in enumerate(ids)}
    return slo_report_arrays(ids, [idx[r.model_id] for r in records], [r.arrival_ms for r in records],
                             [r.completion_ms for r in records], [r.slo_met for r in records], warmup_fraction)


REQUEST_CSV_HEADER = ["request_id", "model_id", "arrival_ms", "dispatch_ms", "completion_ms", "latency_ms",
                      "queueing_ms", "slo_met"]


def request_csv_rows(records):
    for r in records:
        yield [r.request_id, r.model_id, repr(r.arrival_ms), repr(r.dispatch_ms), repr(r.completion_ms),
               repr(r.latency_ms), repr(r.queueing_ms), int(r.slo_met)]


REPORT_CSV_HEADER = ["model_id", "n_requests", "slo_satisfaction", "p50_latency_ms", "p95_latency_ms",
                     "p99_latency_ms"]


def report_csv_rows(report: dict):
    for mid in sorted(report):
        r = report[mid]
        yield [r.model_id, r.n_requests, repr(r.slo_satisfaction), repr(r.p50_latency_ms), repr(r.p95_latency_ms),
               repr(r.p99_latency_ms)]
