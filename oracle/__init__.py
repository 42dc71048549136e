"""CPU oracle for the intfsim hot path.

TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import this package.  The product path
(`paper_2512_18725_b200`) never imports it and fails loudly without its CUDA
library.

Two layers:
* `liboracle.so` (intf_oracle.c): C restatement of the scheduler replay
  (`simcore.py:103-310` as a literal binary-heap event loop), arrivals
  (`workload.py:74-104`), the noise draw (`oracle.py:24-33`: numpy
  SeedSequence/PCG64/ziggurat + glibc exp/log1p FMA variants) and features.
* numpy restatements below of the predictor/refit/eval math
  (`predict.py:43-205`), feature modes (`colocation.py:46-105`) and metrics
  (`metrics.py:28-79`), each citing the reference line it follows.

Pinned against tests/golden/*.npz, which tests/golden/make_golden.py produced
by running the unmodified reference in the build container.

All scenario inputs use the reference's own JSON scenario dict
(`workload.py:192-218`, `scenario_to_dict`) plus a flattened profile table
`(models, max_bs, solo[rows], thr[rows,3])`, row = model_index*max_bs + bs-1.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import zlib
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

D = ctypes.c_double
I = ctypes.c_int
PD = ctypes.POINTER(ctypes.c_double)
PI = ctypes.POINTER(ctypes.c_int)


class ScenarioIn(ctypes.Structure):
    _fields_ = [
        ("n_models", I), ("rate_rps", PD), ("slo_ms", PD), ("crc", ctypes.POINTER(ctypes.c_uint32)),
        ("name_rank", PI), ("entry_base", PI), ("tab_solo", PD), ("tab_thr", PD),
        ("duration_s", D), ("window_ms", D), ("sigma", D), ("beta", D * 3),
        ("max_bs", I), ("cap", I), ("seed", ctypes.c_uint64), ("oracle_seed", ctypes.c_uint64),
        ("batch_id_base", ctypes.c_uint64),
    ]


class ReplayOut(ctypes.Structure):
    _fields_ = [
        ("b_model", PI), ("b_size", PI), ("b_first_req", PI),
        ("b_formed", PD), ("b_start", PD), ("b_completion", PD), ("b_measured", PD), ("b_profiled", PD),
        ("b_seg_off", PI), ("b_nseg", PI), ("b_done_rank", PI), ("b_running", PI),
        ("s_tbegin", PD), ("s_tend", PD), ("s_slowdown", PD), ("s_colo", PD),
        ("r_batch", PI), ("r_slo_met", ctypes.POINTER(ctypes.c_ubyte)),
        ("cap_batches", I), ("cap_segments", I),
        ("n_batches", I), ("n_segments", I), ("n_reseats", I), ("status", I),
    ]


def build() -> str:
    """Compile liboracle.so (gcc, -ffp-contract=off) if missing or stale."""
    src = os.path.join(_HERE, "intf_oracle.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        for name, res, args in [
            ("oracle_exp", D, [D]),
            ("oracle_log1p", D, [D]),
            ("oracle_noise_draw", D, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, D]),
            ("oracle_ddot", D, [PD, PD, I]),
            ("oracle_random_doubles", None, [ctypes.POINTER(ctypes.c_uint32), I, PD, I]),
            ("oracle_standard_normals", None, [ctypes.POINTER(ctypes.c_uint32), I, PD, I]),
            ("oracle_generate_arrivals", I, [ctypes.POINTER(ScenarioIn), PD, PI, I]),
            ("oracle_run_scenario", I, [ctypes.POINTER(ScenarioIn), PD, PI, I, ctypes.POINTER(ReplayOut)]),
            ("oracle_crc32", ctypes.c_uint32, [ctypes.c_char_p, ctypes.c_size_t]),
        ]:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a, t=PD):
    return a.ctypes.data_as(t)


# ----------------------------------------------------------------- tables
@dataclass
class TableArrays:
    models: list
    max_bs: int
    solo: np.ndarray  # [rows]
    thr: np.ndarray  # [rows, 3]

    def row(self, model_id: str, bs: int) -> int:
        return self.models.index(model_id) * self.max_bs + bs - 1


def table_from_reference_like(table) -> TableArrays:
    """Flatten any object with the reference ProfileTable shape
    (`profiles.py:56-66`: .models(), .max_batch_size, .get(m, bs))."""
    models = list(table.models())
    mbs = int(table.max_batch_size)
    solo = np.zeros(len(models) * mbs)
    thr = np.zeros((len(models) * mbs, 3))
    for mi, m in enumerate(models):
        for bs in range(1, mbs + 1):
            p = table.get(m, bs)
            solo[mi * mbs + bs - 1] = p.solo_duration_ms
            thr[mi * mbs + bs - 1] = (p.l2_throughput, p.dram_throughput, p.sm_throughput)
    return TableArrays(models, mbs, solo, thr)


# --------------------------------------------------------------- scenario
class _Keep:
    """Holds numpy buffers alive for the lifetime of a ctypes struct."""


def scenario_in(spec: dict, tab: TableArrays):
    """Flatten a scenario dict (`workload.py:192-218` layout) for the C oracle."""
    dep = spec["deployed"]
    names = [d["model_id"] for d in dep]
    k = _Keep()
    k.rate = np.array([float(d["arrival_rate_rps"]) for d in dep])
    k.slo = np.array([float(d["slo_ms"]) for d in dep])
    k.crc = np.array([zlib.crc32(n.encode("utf-8")) for n in names], dtype=np.uint32)
    order = sorted(range(len(names)), key=lambda i: names[i])
    k.rank = np.zeros(len(names), dtype=np.int32)
    for r, i in enumerate(order):
        k.rank[i] = r
    k.base = np.array([tab.models.index(n) * tab.max_bs for n in names], dtype=np.int32)
    k.solo = np.ascontiguousarray(tab.solo, dtype=np.float64)
    k.thr = np.ascontiguousarray(tab.thr, dtype=np.float64).reshape(-1)
    orc = spec.get("oracle", {})
    s = ScenarioIn()
    s.n_models = len(names)
    s.rate_rps, s.slo_ms = _p(k.rate), _p(k.slo)
    s.crc = _p(k.crc, ctypes.POINTER(ctypes.c_uint32))
    s.name_rank, s.entry_base = _p(k.rank, PI), _p(k.base, PI)
    s.tab_solo, s.tab_thr = _p(k.solo), _p(k.thr)
    s.duration_s = float(spec["duration_s"])
    s.window_ms = float(spec.get("batching_window_ms", 2.0))
    s.sigma = float(orc.get("noise_sigma", 0.05))
    s.beta = (D * 3)(float(orc.get("beta_l2", 1.0)), float(orc.get("beta_dram", 1.5)), float(orc.get("beta_sm", 0.5)))
    s.max_bs = int(spec.get("max_batch_size", 8))
    s.cap = int(spec.get("concurrency_cap", 2))
    s.seed = int(spec.get("seed", 0))
    s.oracle_seed = int(orc.get("seed", 0))
    s.batch_id_base = int(spec.get("batch_id_base", 0))
    k.struct = s
    return k


def generate_arrivals(spec: dict, tab: TableArrays):
    """`workload.py:74-104` -> (arrival_t f64[n], deployed-model index i32[n])."""
    k = scenario_in(spec, tab)
    cap = 1 << 16
    while True:
        t = np.zeros(cap)
        m = np.zeros(cap, dtype=np.int32)
        n = lib().oracle_generate_arrivals(ctypes.byref(k.struct), _p(t), _p(m, PI), cap)
        if n >= 0:
            return t[:n].copy(), m[:n].copy()
        cap *= 4


SIM_ERRORS = {1: "event scheduled in the past", 2: "dispatch at concurrency cap", 4: "progress != work",
              8: "simulation drained its event queue before quiescence", 16: "output capacity exceeded"}


def run_scenario(spec: dict, tab: TableArrays, arrivals=None) -> dict:
    """`simcore.py:218-310` -> dict of arrays.

    Batches are indexed by batch_id; `order` lists batch ids in the
    reference's outcome order (completion, batch_id) (`simcore.py:305`);
    segments of batch b are seg[b_seg_off[b] : b_seg_off[b]+b_nseg[b]].
    """
    k = scenario_in(spec, tab)
    if arrivals is None:
        arrivals = generate_arrivals(spec, tab)
    t, m = arrivals
    t = np.ascontiguousarray(t, dtype=np.float64)
    m = np.ascontiguousarray(m, dtype=np.int32)
    n = len(t)
    cap_b = max(n, 1)
    cap_s = cap_b * (2 * k.struct.cap - 1) + 1
    o = ReplayOut()
    buf = {}
    for name, dt, size in [
        ("b_model", np.int32, cap_b), ("b_size", np.int32, cap_b), ("b_first_req", np.int32, cap_b),
        ("b_formed", np.float64, cap_b), ("b_start", np.float64, cap_b), ("b_completion", np.float64, cap_b),
        ("b_measured", np.float64, cap_b), ("b_profiled", np.float64, cap_b), ("b_seg_off", np.int32, cap_b),
        ("b_nseg", np.int32, cap_b), ("b_done_rank", np.int32, cap_b), ("b_running", np.int32, cap_b),
        ("s_tbegin", np.float64, cap_s), ("s_tend", np.float64, cap_s), ("s_slowdown", np.float64, cap_s),
        ("s_colo", np.float64, 3 * cap_s), ("r_batch", np.int32, max(n, 1)), ("r_slo_met", np.uint8, max(n, 1)),
    ]:
        a = np.zeros(size, dtype=dt)
        buf[name] = a
        ptype = PD if dt == np.float64 else (PI if dt == np.int32 else ctypes.POINTER(ctypes.c_ubyte))
        setattr(o, name, _p(a, ptype))
    o.cap_batches, o.cap_segments = cap_b, cap_s
    st = lib().oracle_run_scenario(ctypes.byref(k.struct), _p(t), _p(m, PI), n, ctypes.byref(o))
    nb, ns = o.n_batches, o.n_segments
    out = {key: v[:nb].copy() for key, v in buf.items() if key.startswith("b_")}
    for key in ("s_tbegin", "s_tend", "s_slowdown"):
        out[key] = buf[key][:ns].copy()
    out["s_colo"] = buf["s_colo"][: 3 * ns].reshape(ns, 3).copy()
    out["r_batch"] = buf["r_batch"][:n].copy()
    out["r_slo_met"] = buf["r_slo_met"][:n].copy()
    out["arr_t"], out["arr_model"] = t, m
    out["order"] = np.lexsort((np.arange(nb), out["b_completion"]))
    out.update(n_batches=nb, n_segments=ns, n_reseats=o.n_reseats, status=st)
    return out


def noise_draw(seed: int, batch_id: int, seg_idx: int, sigma: float) -> float:
    return lib().oracle_noise_draw(seed, batch_id, seg_idx, sigma)


def c_exp(x: float) -> float:
    return lib().oracle_exp(x)


def c_log1p(x: float) -> float:
    return lib().oracle_log1p(x)


def random_doubles(words, n):
    w = np.ascontiguousarray(words, dtype=np.uint32)
    out = np.zeros(n)
    lib().oracle_random_doubles(_p(w, ctypes.POINTER(ctypes.c_uint32)), len(w), _p(out), n)
    return out


def standard_normals(words, n):
    w = np.ascontiguousarray(words, dtype=np.uint32)
    out = np.zeros(n)
    lib().oracle_standard_normals(_p(w, ctypes.POINTER(ctypes.c_uint32)), len(w), _p(out), n)
    return out


def int_words(*vals) -> np.ndarray:
    """numpy SeedSequence entropy coercion (`_int_to_uint32_array`)."""
    w = []
    for v in vals:
        v = int(v)
        if v == 0:
            w.append(0)
        while v > 0:
            w.append(v & 0xFFFFFFFF)
            v >>= 32
    return np.array(w, dtype=np.uint32)


# ------------------------------------------------------------ features (numpy)
def features(colo_hist: np.ndarray, own: np.ndarray, ewma: bool, alpha: float) -> np.ndarray:
    """estimate_from_history + finalize_features (`colocation.py:54-84`)."""
    r = np.array(colo_hist[0], dtype=float)
    if ewma:
        for x_t in colo_hist[1:]:
            r = alpha * np.asarray(x_t, dtype=float) + (1.0 - alpha) * r  # `colocation.py:61`
    return np.concatenate([np.asarray(own, dtype=float), r])


def samples_from_replay(rep: dict, spec: dict, tab: TableArrays, ewma: bool, alpha: float):
    """samples_from_outcomes (`colocation.py:95-105`) over oracle replay arrays,
    in outcome order. Returns (X[n,6], y[n], batch_ids[n])."""
    names = [d["model_id"] for d in spec["deployed"]]
    X, y = [], []
    for b in rep["order"]:
        row = tab.row(names[rep["b_model"][b]], int(rep["b_size"][b]))
        off, ns = rep["b_seg_off"][b], rep["b_nseg"][b]
        X.append(features(rep["s_colo"][off : off + ns], tab.thr[row], ewma, alpha))
        y.append(rep["b_measured"][b] / rep["b_profiled"][b])  # `simcore.py:83-85`
    return np.array(X).reshape(-1, 6), np.array(y), rep["order"].copy()


# ------------------------------------------------------------ predictor (numpy)
RIDGE_EPS = 1e-8  # `predict.py:18`
P_RESET_DELTA = 100.0  # `predict.py:19`


def predict(w, b, x) -> float:
    """`predict.py:43-44`: w @ x + b (BLAS ddot)."""
    return float(np.asarray(w, dtype=float) @ np.asarray(x, dtype=float) + b)


def gram_rows(Z):
    """Z^T Z summed row by row in order: an equally valid summation order to
    BLAS's blocked dgemm, used to measure how far the reference's own result
    moves under reordering when Z^T Z is (nearly) singular."""
    G = np.zeros((Z.shape[1], Z.shape[1]))
    for z in Z:
        G = G + np.outer(z, z)
    return G


def fit_ols_xy(X, y, gram=None):
    """`predict.py:53-66`: lstsq with intercept; ridge fallback if rank-deficient.
    gram: optional Z -> Z^T Z (default numpy's Z.T @ Z)."""
    X = np.asarray(X, dtype=float)
    n, d = X.shape
    Z = np.column_stack([X, np.ones(n)])
    if np.linalg.matrix_rank(Z) < d + 1:
        G = (gram(Z) if gram else Z.T @ Z) + RIDGE_EPS * np.eye(d + 1)
        params = np.linalg.solve(G, Z.T @ y)
    else:
        params, *_ = np.linalg.lstsq(Z, y, rcond=None)
    return params[:d].copy(), float(params[d])


def sgd_update(w, b, x, y, eta):
    """`predict.py:88-95` (returns new (w, b))."""
    x = np.asarray(x, dtype=float)
    e = y - predict(w, b, x)
    w = w + eta * e * x
    b = b + eta * e
    return w, b


def rls_init_P(X_train=None, d=7, delta=P_RESET_DELTA, gram=None):
    """`predict.py:112-134`: P0 = inv(Z^T Z) (ridge on LinAlgError) or delta*I."""
    if X_train is not None:
        Z = np.column_stack([X_train, np.ones(len(X_train))])
        G = gram(Z) if gram else Z.T @ Z
        try:
            return np.linalg.inv(G)
        except np.linalg.LinAlgError:
            return np.linalg.inv(G + RIDGE_EPS * np.eye(d))
    return delta * np.eye(d)


def rls_update(w, b, P, x, y, lam):
    """`predict.py:137-154` (returns new (w, b, P))."""
    x = np.asarray(x, dtype=float)
    z = np.append(x, 1.0)
    Pz = P @ z
    denom = lam + z @ Pz
    if denom <= 0 or not np.isfinite(denom):
        P = P_RESET_DELTA * np.eye(len(z))
        Pz = P @ z
        denom = lam + z @ Pz
    k = Pz / denom
    e = y - predict(w, b, x)
    w = w + k[:-1] * e
    b = b + float(k[-1]) * e
    P = (P - np.outer(k, Pz)) / lam
    P = 0.5 * (P + P.T)
    return w, b, P


def percentile(values, p: float) -> float:
    """Nearest-rank percentile (`metrics.py:28-36`)."""
    v = sorted(values)
    if not v:
        raise ValueError("percentile of empty list")
    rank = max(1, math.ceil(p / 100.0 * len(v)))
    return v[rank - 1]


def eval_report(y_hat, y):
    """`predict.py:195-205` -> (mse, p25, p50, p75, p95, n)."""
    y_hat = np.asarray(y_hat, dtype=float)
    y = np.asarray(y, dtype=float)
    rel = np.abs(y_hat - y) / y
    return (float(np.mean((y_hat - y) ** 2)), float(percentile(rel, 25)), float(percentile(rel, 50)),
            float(percentile(rel, 75)), float(percentile(rel, 95)), len(y))


def prequential(w, b, X, y, method, eta=0.01, lam=0.99, P=None):
    """`predict.py:157-205` online branch: score then update, in order."""
    w = np.array(w, dtype=float)
    preds = []
    for x_i, y_i in zip(X, y):
        preds.append(predict(w, b, x_i))
        if method == "sgd":
            w, b = sgd_update(w, b, x_i, y_i, eta)
        elif method == "rls":
            w, b, P = rls_update(w, b, P, x_i, y_i, lam)
    return np.array(preds), w, b, P


def slo_report(model_ids, arrival, completion, slo_met, warmup_fraction=0.0):
    """`metrics.py:49-79` -> {model: (n, satisfaction, p50, p95, p99)}."""
    arrival = np.asarray(arrival)
    keep = np.ones(len(arrival), dtype=bool)
    if warmup_fraction:
        t0, t1 = arrival.min(), arrival.max()
        cutoff = t0 + warmup_fraction * (t1 - t0)
        keep = arrival >= cutoff
        if not keep.any():
            keep[:] = True
    out = {}
    ids = np.asarray(model_ids)
    for m in sorted(set(ids[keep].tolist())):
        sel = keep & (ids == m)
        lat = (np.asarray(completion)[sel] - arrival[sel]).tolist()
        met = np.asarray(slo_met)[sel]
        out[m] = (int(sel.sum()), sum(bool(v) for v in met) / int(sel.sum()), percentile(lat, 50),
                  percentile(lat, 95), percentile(lat, 99))
    return out


def scenario_eval(rep: dict, spec: dict, tab: TableArrays, lam: float = 0.99, alpha: float = 0.5, gram=None):
    """C5 per-scenario evaluation composed from the reference's
    functions: samples in outcome order (`colocation.py:95-105`), the
    chronological split cut = int(round(0.75 n)) (`experiments.py:44-60`),
    coarse = fit_ols(static) / fine = fit_ols(EWMA(alpha)) scored offline on
    the tail, adaptive = rls_init(fine, lam, X_train) scored prequentially
    (`predict.py:53-72,112-134,157-205`).  Returns [3][6] reports (mse, p25,
    p50, p75, p95, n) or None when split/fit_ols would raise (< 7 training
    samples or an empty test set)."""
    Xs, y, _ = samples_from_replay(rep, spec, tab, False, 1.0)
    Xf, _, _ = samples_from_replay(rep, spec, tab, True, alpha)
    n = len(y)
    cut = int(round(0.75 * n))
    if cut < 7 or n - cut < 1:
        return None
    wc, bc = fit_ols_xy(Xs[:cut], y[:cut], gram)
    wf, bf = fit_ols_xy(Xf[:cut], y[:cut], gram)
    out = [eval_report(Xs[cut:] @ wc + bc, y[cut:]), eval_report(Xf[cut:] @ wf + bf, y[cut:])]
    preds, _, _, _ = prequential(wf, bf, Xf[cut:], y[cut:], "rls", lam=lam, P=rls_init_P(Xf[:cut], gram=gram))
    out.append(eval_report(preds, y[cut:]))
    return np.array(out)


def drift_experiment(specs4, tab: TableArrays, eta: float = 0.01, lam: float = 0.99, alpha: float = 0.5,
                     max_test: int = 300):
    """`experiments.py:153-205` over the 4 drift scenario dicts (TrainingSet,
    TestSet1..3, EWMA(alpha) features): OLS warm start on the training set,
    its offline training score, then per test set (first max_test samples)
    offline / SGD / RLS (P0 = inv(Z^T Z) of the training design) scores.
    Returns [(dataset, method, mse, n)] in the reference's cell order."""
    data = []
    for k, spec in enumerate(specs4):
        X, y, _ = samples_from_replay(run_scenario(spec, tab), spec, tab, True, alpha)
        if k and max_test:
            X, y = X[:max_test], y[:max_test]
        data.append((X, y))
    (Xt, yt) = data[0]
    w0, b0 = fit_ols_xy(Xt, yt)
    tr = eval_report(Xt @ w0 + b0, yt)
    cells = [("TrainingSet", m, tr[0], tr[5]) for m in ("offline", "sgd", "rls")]
    P0 = rls_init_P(Xt)
    for name, (X, y) in zip(("TestSet1", "TestSet2", "TestSet3"), data[1:]):
        off = eval_report(X @ w0 + b0, y)
        sg = eval_report(prequential(w0, b0, X, y, "sgd", eta=eta)[0], y)
        rl = eval_report(prequential(w0, b0, X, y, "rls", lam=lam, P=P0.copy())[0], y)
        cells += [(name, "offline", off[0], off[5]), (name, "sgd", sg[0], sg[5]), (name, "rls", rl[0], rl[5])]
    return cells


# ------------------------------------------------------ candidate sets (C2)
def candidate_history(own: int, peers, solo: np.ndarray, thr: np.ndarray):
    """Fine-grained candidate history: snapshot with all peers
    (summed in peer order from zeros, `simcore.py:126-131`), then one snapshot
    per peer departure for peers whose solo time is shorter than own's,
    departing in (solo_ms, entry) order."""
    hist = []
    c = np.zeros(3)
    for q in peers:
        c = c + thr[q]
    hist.append(c)
    remaining = list(peers)
    for _, q, _j in sorted((solo[q], q, j) for j, q in enumerate(peers) if solo[q] < solo[own]):
        remaining.remove(q)
        c = np.zeros(3)
        for r in remaining:
            c = c + thr[r]
        hist.append(c)
    return hist


def candidate_predictions(own, peers, solo, thr, w_coarse, w_fine, alpha):
    """(y_coarse, y_fine) for one candidate set: static features -> coarse
    model, EWMA(alpha) features -> fine model (`colocation.py:71-84`,
    `predict.py:43-44`).  w_* = 7-vectors (w0..w5, b)."""
    hist = candidate_history(own, peers, solo, thr)
    xs = features(hist, thr[own], False, 1.0)
    xf = features(hist, thr[own], True, alpha)
    return predict(w_coarse[:6], w_coarse[6], xs), predict(w_fine[:6], w_fine[6], xf)


def multisets(E: int, cap: int) -> np.ndarray:
    """Every peer multiset of size <= cap-1 over E entries, as sorted index
    rows padded with -1, in the product's output order (size-major, colex
    within a size: rank = sum_j C(E+j-1, j) for j < k + sum_i C(p_i+i-1, i))."""
    import itertools

    rows = []
    for k in range(cap):
        combos = (np.array(list(itertools.combinations_with_replacement(range(E), k)), dtype=np.int64)
                  if k else np.zeros((1, 0), dtype=np.int64))
        rank = np.zeros(len(combos), dtype=np.int64)
        for i in range(k):
            rank += np.array([math.comb(int(q) + i, i + 1) for q in combos[:, i]], dtype=np.int64)
        block = np.full((len(combos), cap - 1), -1, dtype=np.int64)
        block[rank, :k] = combos
        rows.append(block)
    return np.concatenate(rows)


def candidate_features_all(solo, thr, cap: int, alpha: float):
    """Vectorised `candidate_history` + `features` for every (own, multiset):
    (X_static, X_ewma) of shape [E, n_sets, 6], fp64.  Peer sums run from
    zeros in peer order (`simcore.py:126-131`); a removed peer contributes an
    exact +0.0, so the sums equal the scalar restatement's bit for bit; the
    EWMA recursion is `colocation.py:61` unfused."""
    solo = np.asarray(solo, dtype=float)
    thr = np.asarray(thr, dtype=float)
    E = len(solo)
    M = multisets(E, cap)  # [n_sets, cap-1]
    k = cap - 1
    valid = M >= 0
    Mi = np.where(valid, M, 0)
    pthr = thr[Mi] * valid[..., None]  # [n, k, 3], zeros for absent peers
    c0 = np.zeros((len(M), 3))
    for j in range(k):
        c0 = c0 + pthr[:, j]
    Xs = np.empty((E, len(M), 6))
    Xf = np.empty((E, len(M), 6))
    psolo = np.where(valid, solo[Mi], np.inf)
    for own in range(E):
        dep = valid & (psolo < solo[own])  # peers that finish before own
        # departure order (solo, entry, position): peers are sorted by entry, so a stable sort by solo is it
        key = np.where(dep, psolo, np.inf)
        order = np.argsort(key, axis=1, kind="stable")
        alive = valid.copy()
        r = c0.copy()
        for t in range(k):
            q = order[:, t]
            has = dep[np.arange(len(M)), q]
            alive[np.arange(len(M))[has], q[has]] = False
            c = np.zeros((len(M), 3))
            for j in range(k):
                c = c + np.where(alive[:, j, None], pthr[:, j], 0.0)
            r = np.where(has[:, None], alpha * c + (1.0 - alpha) * r, r)
        own_x = np.broadcast_to(thr[own], (len(M), 3))
        Xs[own] = np.concatenate([own_x, c0], axis=1)
        Xf[own] = np.concatenate([own_x, r], axis=1)
    return Xs, Xf


def candidate_predictions_all(solo, thr, cap: int, W, alpha: float) -> np.ndarray:
    """Every candidate's (coarse, fine) prediction for every decision:
    [n_dec, 2, E, n_sets] fp64, the product's logical output layout
    (`CandidateScorer.view`).  W = [n_dec][2][7] (w0..w5, b)."""
    Xs, Xf = candidate_features_all(solo, thr, cap, alpha)
    W = np.asarray(W, dtype=float).reshape(-1, 2, 7)
    out = np.empty((len(W), 2, Xs.shape[0], Xs.shape[1]))
    for d in range(len(W)):
        out[d, 0] = Xs @ W[d, 0, :6] + W[d, 0, 6]
        out[d, 1] = Xf @ W[d, 1, :6] + W[d, 1, 6]
    return out


# ------------------------------------------------ calibration driver (§8f)
def _slowdown(own, colo, betas, noise: float) -> float:
    """`oracle.py:36-47`: (1 + betas @ max(0, own + colo - 1)) * noise, the
    dot an fma chain from 0 (OpenBLAS ddot)."""
    excess = np.maximum(0.0, (np.asarray(own, dtype=float) + np.asarray(colo, dtype=float)) - 1.0)
    b = np.ascontiguousarray(betas, dtype=np.float64)
    dot = lib().oracle_ddot(_p(b), _p(np.ascontiguousarray(excess)), 3)
    return (1.0 + dot) * noise


def full_overlap_ratios(tab: TableArrays, model_a="roberta_b", model_b="roberta_b", batch_size=8, n_pairs=200,
                        seed=0, sigma=0.05, betas=(1.0, 1.5, 0.5)):
    """`experiments.py:255-291` restated on GpuState's semantics
    (`simcore.py:103-198`): per pair, batches 2k (model_a) and 2k+1 (model_b)
    dispatched at t = 0 in that order (the second dispatch pops the first
    batch's zero-length segment and reseats it at segment index 0), then
    completions in (remaining * slowdown, batch_id) order, now += that
    product, the survivor reseated alone.  Returns the interference ratios
    in completion order."""
    def noise(b, i):
        return 1.0 if sigma == 0.0 else noise_draw(seed, b, i, sigma)

    out = []
    for k in range(n_pairs):
        ids = (2 * k, 2 * k + 1)
        rows = (tab.row(model_a, batch_size), tab.row(model_b, batch_size))
        own = [np.asarray(tab.thr[r], dtype=float) for r in rows]
        total = [float(tab.solo[r]) for r in rows]
        # dispatch a: alone; dispatch b: b reseated (colo = own_a), a's zero-length segment popped and
        # a reseated with colo = own_b at segment index 0 again
        sd = [_slowdown(own[0], np.zeros(3) + own[1], betas, noise(ids[0], 0)),
              _slowdown(own[1], np.zeros(3) + own[0], betas, noise(ids[1], 0))]
        hist = [[sd[0]], [sd[1]]]
        prog = [0.0, 0.0]
        now = 0.0
        first = min((0, 1), key=lambda j: ((total[j] - prog[j]) * sd[j], ids[j]))
        now += (total[first] - prog[first]) * sd[first]
        order = [first, 1 - first]
        j = first
        prog[j] += (now - 0.0) / sd[j]
        out.append((total[j] if all(s == 1.0 for s in hist[j]) else now - 0.0) / total[j])
        y = 1 - first  # survivor: close its segment [0, now), reseat alone at segment index 1
        prog[y] += (now - 0.0) / sd[y]
        sd[y] = _slowdown(own[y], np.zeros(3), betas, noise(ids[y], 1))
        hist[y].append(sd[y])
        now += (total[y] - prog[y]) * sd[y]
        out.append((total[y] if all(s == 1.0 for s in hist[y]) else now - 0.0) / total[y])
        del order
    return out
