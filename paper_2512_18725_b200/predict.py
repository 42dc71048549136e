"""Linear interference predictor y_hat = w.x + b: offline OLS, online SGD
and RLS, prequential evaluation.  Mirrors `intfsim.predict`
(`predict.py:16-235`).  Every numeric step is a kernel (K6 OLS statistics +
7x7 fp64 solve, K7 prequential streams, K8 eval reduction); the batched
entry points (`fit_ols_many`, `evaluate_many`) are what the experiment
drivers use."""
from __future__ import annotations

import json
import logging
from dataclasses import dataclass
from pathlib import Path

import numpy as np

log = logging.getLogger(__name__)

N_FEATURES = 6
RIDGE_EPS = 1e-8
P_RESET_DELTA = 100.0


class PredictError(RuntimeError):
    """Numerically invalid predictor state (`predict.py:22`)."""


@dataclass
class LinearModel:
    w: np.ndarray
    b: float

    def copy(self) -> "LinearModel":
        return LinearModel(w=self.w.copy(), b=self.b)

    def check_finite(self, context: str = "") -> None:
        if not (np.all(np.isfinite(self.w)) and np.isfinite(self.b)):
            raise PredictError(f"non-finite model parameters {context}")

    def w7(self) -> np.ndarray:
        return np.append(np.asarray(self.w, dtype=float), float(self.b))


def zero_model(n_features: int = N_FEATURES) -> LinearModel:
    return LinearModel(w=np.zeros(n_features), b=0.0)


def predict(model: LinearModel, x) -> float:
    """w @ x + b (`predict.py:43-44`) on the device (fma chain == BLAS ddot)."""
    from . import engine

    return float(engine.scalar(engine.SCALAR_PREDICT, (), np.concatenate([model.w7(),
                                                                        np.asarray(x, dtype=float).reshape(6)]))[0])


def predict_many(model: LinearModel, X) -> np.ndarray:
    from . import engine

    return engine.predict_rows(np.asarray(X, dtype=float).reshape(-1, 6), model.w7())


def _design(samples):
    return (np.array([s.x for s in samples], dtype=float).reshape(-1, 6), np.array([s.y for s in samples], dtype=float))


def fit_ols_xy(X, y) -> LinearModel:
    """Least squares with intercept; ridge fallback if rank-deficient
    (`predict.py:53-66`).  Z^T Z / Z^T y reduced on the device in fp64; an
    ill-conditioned design takes its rank and solution from a device QR of
    its rows."""
    from . import engine

    params, ridge, nonfinite = engine.ols_fit(np.asarray(X, dtype=float), np.asarray(y, dtype=float))
    if ridge:
        log.warning("rank-deficient design matrix (n=%d), using ridge fallback", len(X))
    model = LinearModel(w=params[:6].copy(), b=float(params[6]))
    model.check_finite("after OLS fit")
    return model


def fit_ols(samples) -> LinearModel:
    if len(samples) < N_FEATURES + 1:
        raise PredictError(f"need >= {N_FEATURES + 1} samples, got {len(samples)}")
    return fit_ols_xy(*_design(samples))


def fit_ols_windows(X, y, window: int) -> list:
    """Refit each window: `[fit_ols_xy(X[i:i+window], y[i:i+window]) for i
    in range(0, n, window)]` (`predict.py:53-66`), all windows in one
    statistics launch and one solve launch (a window of fewer than 7 rows is
    rank-deficient and takes the ridge fallback, as in fit_ols_xy)."""
    from . import engine

    X = np.asarray(X, dtype=float).reshape(-1, 6)
    y = np.asarray(y, dtype=float)
    params, info = engine.ols_windows(X, y, int(window))
    out = []
    for k, (p, inf) in enumerate(zip(params, info)):
        if inf[0]:
            log.warning("rank-deficient design matrix (window %d), using ridge fallback", k)
        model = LinearModel(w=p[:6].copy(), b=float(p[6]))
        model.check_finite("after OLS fit")
        out.append(model)
    return out


@dataclass
class SgdState:
    model: LinearModel
    eta: float = 0.01

    def __post_init__(self):
        if not self.eta > 0:
            raise PredictError("eta must be positive")

    def copy(self) -> "SgdState":
        return SgdState(model=self.model.copy(), eta=self.eta)


def _sgd_run(state: SgdState, X, y):
    from . import engine

    preds, params, st = engine.sgd_streams([X], [y], state.model.w7()[None], [state.eta])
    state.model.w[:] = params[0, :6]
    state.model.b = float(params[0, 6])
    if st[0] & 1:
        raise PredictError(f"non-finite model parameters after SGD step (eta={state.eta})")
    return preds[0]


def sgd_update(state: SgdState, sample) -> SgdState:
    """One LMS step (`predict.py:88-95`), in place (one scalar device call)."""
    from . import engine

    out = engine.scalar(engine.SCALAR_SGD, (), np.concatenate([state.model.w7(), np.asarray(sample.x, dtype=float)
                                                               .reshape(6), [float(sample.y), float(state.eta)]]))
    state.model.w[:] = out[:6]
    state.model.b = float(out[6])
    if out[8]:
        raise PredictError(f"non-finite model parameters after SGD step (eta={state.eta})")
    return state


@dataclass
class RlsState:
    model: LinearModel
    P: np.ndarray
    lam: float = 0.99

    def __post_init__(self):
        if not (0.0 < self.lam <= 1.0):
            raise PredictError("forgetting factor must lie in (0, 1]")

    def copy(self) -> "RlsState":
        return RlsState(model=self.model.copy(), P=self.P.copy(), lam=self.lam)


def rls_init(model: LinearModel, lam: float = 0.99, X_train=None, delta: float = P_RESET_DELTA) -> RlsState:
    """P0 = inv(Z^T Z) of the training design, else delta*I (`predict.py:112-134`)."""
    from . import engine

    d = model.w.shape[0] + 1
    if X_train is not None:
        X_train = np.asarray(X_train, dtype=float)
        stats = engine.ols_stats(X_train, np.zeros(len(X_train)))
        _, _, _, P = engine.ols_solve(stats, want_pinv=True)
    else:
        P = delta * np.eye(d)
    return RlsState(model=model.copy(), P=P, lam=lam)


def _rls_run(state: RlsState, X, y):
    from . import engine

    preds, params, P, st = engine.rls_streams([X], [y], state.model.w7()[None], state.P[None], [state.lam])
    if st[0] & 2:
        log.warning("RLS gain matrix lost positive-definiteness; resetting P")
    state.model.w[:] = params[0, :6]
    state.model.b = float(params[0, 6])
    state.P = P[0]
    if st[0] & 1:
        raise PredictError("non-finite model parameters after RLS step")
    return preds[0]


def rls_update(state: RlsState, sample) -> RlsState:
    """`predict.py:137-154`, in place (one scalar device call)."""
    from . import engine

    out = engine.scalar(engine.SCALAR_RLS, (), np.concatenate([state.model.w7(), np.asarray(state.P, dtype=float)
                                                               .reshape(49), np.asarray(sample.x, dtype=float)
                                                               .reshape(6), [float(sample.y), float(state.lam)]]))
    st = int(out[57])
    if st & 2:
        log.warning("RLS gain matrix lost positive-definiteness; resetting P")
    state.model.w[:] = out[:6]
    state.model.b = float(out[6])
    state.P = out[7:56].reshape(7, 7).copy()
    if st & 1:
        raise PredictError("non-finite model parameters after RLS step")
    return state


def score_and_update(predictor, sample) -> float:
    """Prequential step: pre-update prediction, then learn (`predict.py:157-172`)."""
    x = np.asarray(sample.x, dtype=float)[None]
    if isinstance(predictor, LinearModel):
        return predict(predictor, sample.x)
    if isinstance(predictor, SgdState):
        return float(_sgd_run(predictor, x, [sample.y])[0])
    if isinstance(predictor, RlsState):
        return float(_rls_run(predictor, x, [sample.y])[0])
    raise TypeError(f"unknown predictor type {type(predictor)!r}")


@dataclass(frozen=True)
class EvalReport:
    mse: float
    rel_p25: float
    rel_p50: float
    rel_p75: float
    rel_p95: float
    n_samples: int


def _report(row) -> EvalReport:
    return EvalReport(float(row[0]), float(row[1]), float(row[2]), float(row[3]), float(row[4]), int(row[5]))


def evaluate(predictor, samples, online: bool = False) -> EvalReport:
    """Score in order; online = prequential (`predict.py:185-205`)."""
    if not samples:
        raise PredictError("evaluate on empty sample list")
    return evaluate_many([predictor], [samples], online=online)[0]


def evaluate_many(predictors, datasets, online: bool = False) -> list:
    """Batched evaluate: one device stream per (predictor, dataset) pair, all
    launched together; SGD/RLS states are updated in place."""
    from . import engine

    Xs, ys = zip(*[_design(s) for s in datasets])
    yhats = [None] * len(predictors)
    if online:
        sgd = [i for i, p in enumerate(predictors) if isinstance(p, SgdState)]
        rls = [i for i, p in enumerate(predictors) if isinstance(p, RlsState)]
        if sgd:
            pr, params, st = engine.sgd_streams([Xs[i] for i in sgd], [ys[i] for i in sgd],
                                                np.stack([predictors[i].model.w7() for i in sgd]),
                                                [predictors[i].eta for i in sgd])
            for j, i in enumerate(sgd):
                predictors[i].model.w[:] = params[j, :6]
                predictors[i].model.b = float(params[j, 6])
                if st[j] & 1:
                    raise PredictError(f"non-finite model parameters after SGD step (eta={predictors[i].eta})")
                yhats[i] = pr[j]
        if rls:
            pr, params, P, st = engine.rls_streams([Xs[i] for i in rls], [ys[i] for i in rls],
                                                   np.stack([predictors[i].model.w7() for i in rls]),
                                                   np.stack([predictors[i].P for i in rls]),
                                                   [predictors[i].lam for i in rls])
            for j, i in enumerate(rls):
                if st[j] & 2:
                    log.warning("RLS gain matrix lost positive-definiteness; resetting P")
                predictors[i].model.w[:] = params[j, :6]
                predictors[i].model.b = float(params[j, 6])
                predictors[i].P = P[j]
                if st[j] & 1:
                    raise PredictError("non-finite model parameters after RLS step")
                yhats[i] = pr[j]
    for i, p in enumerate(predictors):
        if yhats[i] is None:
            model = p if isinstance(p, LinearModel) else p.model
            if not isinstance(p, (LinearModel, SgdState, RlsState)):
                raise TypeError(f"unknown predictor type {type(p)!r}")
            yhats[i] = engine.predict_rows(Xs[i], model.w7())
    rows = engine.eval_reports(yhats, ys)
    return [_report(r) for r in rows]


EVAL_CSV_HEADER = ["dataset", "method", "mse", "rel_p25", "rel_p50", "rel_p75", "rel_p95", "n_samples"]


def save_model(model: LinearModel, path) -> None:
    Path(path).write_text(json.dumps({"w": model.w.tolist(), "b": model.b}, indent=2) + "\n", encoding="utf-8")


def load_model(path) -> LinearModel:
    data = json.loads(Path(path).read_text(encoding="utf-8"))
    return LinearModel(w=np.array(data["w"], dtype=float), b=float(data["b"]))
