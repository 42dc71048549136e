"""Co-location features: static dispatch snapshot vs EWMA over co-location
changes.  Mirrors `intfsim.colocation` (`colocation.py:11-126`).

The per-estimate helpers fold histories on the GPU with the same kernel as
the batched `samples_from_outcomes` (one sample per outcome, K4/K5)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

STATIC = "static"
EWMA = "ewma"


@dataclass(frozen=True)
class Mode:
    kind: str
    alpha: float = 1.0

    def __post_init__(self):
        if self.kind not in (STATIC, EWMA):
            raise ValueError(f"unknown co-location mode {self.kind!r}")
        if self.kind == EWMA and not (0.0 < self.alpha <= 1.0):
            raise ValueError(f"alpha {self.alpha} outside (0, 1]")

    def label(self) -> str:
        return "static" if self.kind == STATIC else f"ewma_{self.alpha:.4g}"

    def predictor(self, w7=(0.0,) * 7):
        """C-ABI predictor block for this mode (w0..w5, b)."""
        from ._abi import Predictor

        return Predictor(ewma=int(self.kind == EWMA), alpha=float(self.alpha), w=tuple(float(v) for v in w7))


STATIC_MODE = Mode(STATIC)


def ewma_mode(alpha: float) -> Mode:
    return Mode(EWMA, alpha)


@dataclass
class CoLocationEstimate:
    batch_id: int
    mode: Mode
    r_hat: np.ndarray
    n_observations: int = 1


def _check_nonneg(v):
    v = np.asarray(v, dtype=float)
    if np.any(v < 0):
        raise ValueError(f"negative co-location throughput: {v}")
    return v


def _fold(history: np.ndarray, mode: Mode) -> np.ndarray:
    """EWMA / static fold of a [k,3] history on the device."""
    from . import engine

    h = np.asarray(history, dtype=float).reshape(-1, 3)
    _, _, yhat = engine.features_rows(np.zeros((1, 3)), np.array([0]), np.array([len(h)]), h, np.ones(1), np.ones(1),
                                      [mode.predictor((0, 0, 0, 1, 0, 0, 0)), mode.predictor((0, 0, 0, 0, 1, 0, 0)),
                                       mode.predictor((0, 0, 0, 0, 0, 1, 0))], want_x=False)
    return yhat[:, 0].copy()


def init_estimate(batch_id: int, mode: Mode, colo_now) -> CoLocationEstimate:
    """Dispatch-time snapshot (`colocation.py:46-51`)."""
    return CoLocationEstimate(batch_id=batch_id, mode=mode, r_hat=_check_nonneg(colo_now).copy())


def observe(est: CoLocationEstimate, x_t) -> CoLocationEstimate:
    """One co-location change (`colocation.py:54-63`); no-op in static mode."""
    x_t = _check_nonneg(x_t)
    if est.mode.kind == EWMA:
        from . import engine

        est.r_hat = engine.scalar(engine.SCALAR_EWMA, (), np.concatenate([np.asarray(est.r_hat, dtype=float)
                                                                          .reshape(3), x_t.reshape(3),
                                                                          [float(est.mode.alpha)]]))
        est.n_observations += 1
    return est


def finalize_features(profile, est: CoLocationEstimate) -> np.ndarray:
    return np.concatenate([profile.throughputs(), est.r_hat])


def estimate_from_history(batch_id: int, mode: Mode, history) -> CoLocationEstimate:
    """Fold a recorded colo history (`colocation.py:71-84`)."""
    if len(history) == 0:
        raise ValueError("empty co-location history")
    h = np.asarray([_check_nonneg(x) for x in history], dtype=float)
    r = h[0].copy() if mode.kind == STATIC else _fold(h, mode)
    return CoLocationEstimate(batch_id=batch_id, mode=mode, r_hat=r, n_observations=len(h) if mode.kind == EWMA else 1)


@dataclass(frozen=True)
class Sample:
    x: np.ndarray
    y: float
    batch_id: int
    scenario: str = ""


def outcome_arrays(outcomes, table):
    """Flatten outcome objects (or reuse the replay arrays) for the device."""
    arrs = getattr(outcomes, "arrays", None)
    if arrs is not None:
        return arrs
    own, off, ns, colo, meas, prof, bids = [], [], [], [], [], [], []
    k = 0
    for o in outcomes:
        own.append(table.get(o.model_id, o.batch_size).throughputs())
        h = o.colo_history
        off.append(k)
        ns.append(len(h))
        colo.extend(h)
        k += len(h)
        meas.append(o.measured_duration_ms)
        prof.append(o.profiled_ms)
        bids.append(o.batch_id)
    return {
        "own": np.asarray(own, dtype=float).reshape(-1, 3), "seg_off": np.asarray(off, dtype=np.int64),
        "nseg": np.asarray(ns, dtype=np.int32), "colo": np.asarray(colo, dtype=float).reshape(-1, 3),
        "measured": np.asarray(meas, dtype=float), "profiled": np.asarray(prof, dtype=float),
        "batch_id": np.asarray(bids, dtype=np.int64),
    }


def features_for_modes(outcomes, table, modes):
    """(X[len(modes)][n][6], y[n]) for several feature modes in one launch."""
    from . import engine

    a = outcome_arrays(outcomes, table)
    if len(a["nseg"]) == 0:
        return np.zeros((len(modes), 0, 6)), np.zeros(0), a
    X, y, _ = engine.features_rows(a["own"], a["seg_off"], a["nseg"], a["colo"], a["measured"], a["profiled"],
                                   [m.predictor() for m in modes])
    return X, y, a


def samples_from_outcomes(outcomes, table, mode: Mode, scenario: str = "") -> list:
    """One Sample per completed batch, in outcome order (`colocation.py:95-105`)."""
    X, y, a = features_for_modes(outcomes, table, [mode])
    Xs = np.array(X[0], dtype=float)  # private copy: every Sample views its own row
    ys, bids = np.asarray(y, dtype=float).tolist(), np.asarray(a["batch_id"]).tolist()
    return [Sample(x=Xs[i], y=ys[i], batch_id=bids[i], scenario=scenario) for i in range(len(ys))]


SAMPLE_CSV_HEADER = ["batch_id", "scenario", "own_l2", "own_dram", "own_sm", "colo_l2", "colo_dram", "colo_sm",
                     "y_ratio", "mode", "alpha"]


def sample_csv_rows(samples, mode: Mode):
    alpha = mode.alpha if mode.kind == EWMA else ""
    for s in samples:
        yield [s.batch_id, s.scenario, *["%r" % v for v in s.x], repr(s.y), mode.kind, alpha]
