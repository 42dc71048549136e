"""Device pipeline driver: scenarios -> (arrivals -> replay -> SLO ->
features/predict) on the current CUDA device, through the C ABI.

torch is used only for device memory and the current stream; every
computation is a kernel in libintfsim_b200.so.  Without a CUDA device the
constructor raises -- there is no CPU path.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _abi, _pack

_TORCH_DT = {np.float64: torch.float64, np.int32: torch.int32, np.uint8: torch.uint8, np.float32: torch.float32,
             np.int64: torch.int64}
_NP_DT = {v: np.dtype(k) for k, v in _TORCH_DT.items()}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2512_18725_b200: a CUDA (sm_100a) device is required; the hot path has no CPU implementation"
        )
    _abi.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def to_device(a: np.ndarray, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=False)


def _struct_bytes(arr) -> np.ndarray:
    return np.frombuffer(bytes(arr), dtype=np.uint8).copy()


class DeviceTable:
    """Profile table resident in HBM (`profiles.py:56-66`)."""

    def __init__(self, table: _pack.TableArrays, dev=None):
        dev = dev or require_cuda()
        self.host = table
        self.solo = to_device(np.asarray(table.solo, dtype=np.float64), dev)
        self.thr = to_device(np.asarray(table.thr, dtype=np.float64).reshape(-1), dev)
        self.struct = _abi.Table(self.solo.data_ptr(), self.thr.data_ptr(), len(table.solo), int(table.max_bs))


NOISE_K = 6  # noise draws precomputed per batch (measured best: profiles/noise_k_r1m.txt)


class ReplayPipeline:
    """Buffers + launches for one packed batch of scenarios.

    `run()` only enqueues kernels on the current stream (no host sync), so a
    step can be timed with CUDA events or captured in a CUDA graph.
    """

    def __init__(self, specs, table: _pack.TableArrays, seg_stride: int = 64, scale: float = 1.0,
                 preds=(), list_caps=None, dtable: DeviceTable | None = None, noise_k: int | None = None,
                 evaluate=None):
        self.dev = require_cuda()
        self.lib = _abi.load()
        self.pb = _pack.pack(list(specs), table, scale=scale, list_caps=list_caps)
        self.seg_stride = int(seg_stride)
        self.dtable = dtable or DeviceTable(table, self.dev)
        # noise draws precomputed per batch (the rest are drawn on the replay chain)
        self.noise_k = int(noise_k if noise_k is not None else NOISE_K)
        sz = _pack.sizes(self.pb, self.seg_stride, self.noise_k)
        self.t = {f: torch.zeros(sz[k], dtype=_TORCH_DT[dt], device=self.dev) for f, dt, k in _pack.BUFFER_PLAN}
        self.B = _abi.ReplayBuffers()
        for f in _abi.REPLAY_BUFFER_FIELDS:
            setattr(self.B, f, self.t[f].data_ptr())
        self.B.seg_stride, self.B.cap_max, self.B.noise_k = self.seg_stride, self.pb.cap_max, self.noise_k
        self.d_scen = to_device(_struct_bytes(self.pb.scen), self.dev)
        self.d_models = to_device(_struct_bytes(self.pb.models), self.dev)
        # (model, chunk) of every 256-entry chunk of the long lists: flat grids for their formation
        long_list = int(self.lib.intf_long_list())  # the library's INTF_LONG_LIST
        blk = [(g, c) for g in range(self.pb.n_models) if self.pb.models[g].list_cap >= long_list
               for c in range((self.pb.models[g].list_cap + 255) // 256)]
        self.d_long_blocks = (torch.tensor(blk, dtype=torch.int32).reshape(-1).to(self.dev) if blk else None)
        self.batch = _abi.Batch(self.d_scen.data_ptr(), self.d_models.data_ptr(), self.pb.n_scen, self.pb.n_models,
                                self.pb.max_req_cap, max((len(n) for n in self.pb.names), default=0),
                                max((self.pb.models[g].list_cap for g in range(self.pb.n_models)), default=0),
                                self.pb.total_req, _abi.addr(self.d_long_blocks), len(blk), 0)
        n_models = max(self.pb.n_models, 1)
        self.slo_n = torch.zeros(n_models, dtype=torch.int32, device=self.dev)
        self.slo_met = torch.zeros(n_models, dtype=torch.int32, device=self.dev)
        self.slo_p = torch.zeros(n_models * 3, dtype=torch.float64, device=self.dev)
        self.set_predictors(preds)
        # per-scenario coarse / fine / adaptive evaluation (intf_scenario_eval):
        # evaluate = (p_static, p_ewma, lam) -- indices of the static and EWMA
        # feature modes among `preds`
        self.evaluate = tuple(evaluate) if evaluate is not None else None
        if self.evaluate is not None:
            p_s, p_e, _ = self.evaluate
            if not (0 <= p_s < len(self.preds) and 0 <= p_e < len(self.preds)) or self.preds[p_s].ewma \
                    or not self.preds[p_e].ewma:
                raise ValueError("evaluate=(p_static, p_ewma, lam) must name a static and an EWMA predictor")
            S = max(self.pb.n_scen, 1)
            n_ws = int(self.lib.intf_scenario_eval_ws(S, self.slot_stride))
            self.eval_ws = torch.zeros(n_ws, dtype=torch.float64, device=self.dev)
            self.eval_params = torch.zeros(S * 21, dtype=torch.float64, device=self.dev)
            self.eval_report = torch.zeros(S * 18, dtype=torch.float64, device=self.dev)
            self.eval_status = torch.zeros(2 * S, dtype=torch.int32, device=self.dev)

    # ------------------------------------------------------------ inputs
    def set_predictors(self, preds):
        self.preds = list(preds)
        n = len(self.preds)
        stride = _pack.sizes(self.pb, 1)["req"]
        self.slot_stride = stride
        self.Y = torch.zeros(stride, dtype=torch.float64, device=self.dev)
        self.Yhat = torch.zeros(max(n, 1) * stride, dtype=torch.float64, device=self.dev)
        self.X = torch.zeros(max(n, 1) * stride * 6, dtype=torch.float64, device=self.dev)
        self.P = (_abi.Predictor * max(n, 1))(*self.preds) if n else None

    def load_arrivals(self, arr_t_list, arr_model_list):
        """Caller-supplied merged arrivals (one pair of arrays per scenario)."""
        t = self.t
        n_req = np.zeros(self.pb.n_scen, dtype=np.int32)
        at = np.zeros(t["arr_t"].numel())
        am = np.zeros(t["arr_model"].numel(), dtype=np.int32)
        for s, (tt, mm) in enumerate(zip(arr_t_list, arr_model_list)):
            S = self.pb.scen[s]
            if len(tt) > S.req_cap:
                raise ValueError("arrivals exceed the packed request capacity")
            at[S.req_off:S.req_off + len(tt)] = tt
            am[S.req_off:S.req_off + len(tt)] = mm
            n_req[s] = len(tt)
        t["arr_t"].copy_(torch.from_numpy(at))
        t["arr_model"].copy_(torch.from_numpy(am))
        t["n_req"][: self.pb.n_scen].copy_(torch.from_numpy(n_req))

    # ------------------------------------------------------------ launches
    def run(self, arrivals: bool = True, slo: bool = True, features: bool = True, warm_cutoff=None):
        L, s = self.lib, stream_ptr()
        bt, B = ctypes.byref(self.batch), ctypes.byref(self.B)
        if arrivals:
            _abi.check(L.intf_generate_arrivals(bt, B, s), "intf_generate_arrivals")
        else:
            _abi.check(L.intf_split_arrivals(bt, B, s), "intf_split_arrivals")
        _abi.check(L.intf_replay(bt, ctypes.byref(self.dtable.struct), B, s), "intf_replay")
        self.run_slo_features(warm_cutoff, slo=slo, features=features)

    def run_slo_features(self, warm_cutoff=None, slo: bool = True, features: bool = True, evaluate: bool = True):
        L, s = self.lib, stream_ptr()
        bt, B = ctypes.byref(self.batch), ctypes.byref(self.B)
        if slo:
            _abi.check(L.intf_slo_report(bt, B, _abi.addr(warm_cutoff), self.slo_n.data_ptr(),
                                         self.slo_met.data_ptr(), self.slo_p.data_ptr(), s), "intf_slo_report")
        if features:
            n = len(self.preds)
            _abi.check(L.intf_features_predict(bt, ctypes.byref(self.dtable.struct), B,
                                               ctypes.cast(self.P, ctypes.c_void_p) if n else None, n,
                                               self.slot_stride, self.X.data_ptr(), self.Y.data_ptr(),
                                               self.Yhat.data_ptr(), s), "intf_features_predict")
        if evaluate and self.evaluate is not None:
            self.run_evaluation()

    def run_evaluation(self):
        """Per-scenario coarse / fine / adaptive EvalReports from the features
        of the last run (intf_scenario_eval; enqueue only)."""
        p_s, p_e, lam = self.evaluate
        _abi.check(self.lib.intf_scenario_eval(ctypes.byref(self.batch), ctypes.byref(self.B), self.X.data_ptr(),
                                               self.slot_stride, p_s, p_e, self.Y.data_ptr(), float(lam),
                                               self.eval_ws.data_ptr(), self.eval_ws.numel(),
                                               self.eval_params.data_ptr(), self.eval_report.data_ptr(),
                                               self.eval_status.data_ptr(), stream_ptr()), "intf_scenario_eval")

    def status(self) -> np.ndarray:
        return self.t["status"][: self.pb.n_scen].cpu().numpy()

    # ------------------------------------------------------------ results
    SCRATCH = ("slot_seg", "noise_tab", "mb_t", "mb_info", "n_mb", "slo_ws", "form_ws", "order")

    def fetch(self, scratch: bool = False) -> dict:
        """Copy the result buffers to host numpy (scratch buffers too if asked)
        in ONE device-to-host transfer: the buffers are packed byte-wise on
        the device (stream-ordered copies) and split on the host."""
        src = {k: v for k, v in self.t.items() if scratch or k not in self.SCRATCH}
        src.update(Y=self.Y, Yhat=self.Yhat, X=self.X, slo_n=self.slo_n, slo_met=self.slo_met, slo_p=self.slo_p)
        if self.evaluate is not None:
            src.update(eval_report=self.eval_report, eval_params=self.eval_params, eval_status=self.eval_status)
        parts, offs, off = [], {}, 0
        for k, v in src.items():
            b = v.reshape(-1).view(torch.uint8)
            pad = (-b.numel()) % 8  # keep every buffer 8-byte aligned in the packed copy
            parts.append(b)
            if pad:
                parts.append(torch.zeros(pad, dtype=torch.uint8, device=self.dev))
            offs[k] = (off, v.numel(), v.dtype)
            off += b.numel() + pad
        flat = torch.cat(parts).cpu().numpy()
        h = {k: flat[o:o + n * t.itemsize].view(_NP_DT[t]) for k, (o, n, t) in offs.items()}
        h["Yhat"] = h["Yhat"].reshape(-1, self.slot_stride)
        h["X"] = h["X"].reshape(-1, self.slot_stride, 6)
        h["slo_p"] = h["slo_p"].reshape(-1, 3)
        if self.evaluate is not None:
            h["eval_report"] = h["eval_report"].reshape(-1, 3, 6)
            h["eval_params"] = h["eval_params"].reshape(-1, 3, 7)
            st = h["eval_status"]
            h["eval_status"] = st[: len(st) // 2] | (st[len(st) // 2:] << 8)
        return h

    def scenario(self, h: dict, s: int) -> dict:
        """Per-scenario views of fetched buffers (oracle.run_scenario key layout)."""
        S = self.pb.scen[s]
        ro, n, nb = S.req_off, int(h["n_req"][s]), int(h["n_batches"][s])
        v = {k: h[k][ro:ro + nb] for k in ("b_model", "b_size", "b_formed", "b_start", "b_completion",
                                             "b_measured", "b_seg_off", "b_nseg", "b_running")}
        v["order"] = h["out_order"][ro:ro + nb]
        for k in ("r_batch", "r_slo_met", "arr_t", "arr_model"):
            v[k] = h[k][ro:ro + n]
        for k in ("s_tbegin", "s_tend", "s_slowdown"):
            v[k] = h[k]
        v["s_colo"] = h["s_colo"].reshape(-1, 3)
        v["status"] = int(h["status"][s])
        v["n_reseats"] = int(h["n_reseats"][s])
        v["n_segments"] = int(h["n_segments"][s])
        v["Y"] = h["Y"][ro:ro + nb]
        v["Yhat"] = h["Yhat"][:, ro:ro + nb]
        v["X"] = h["X"][:, ro:ro + nb]
        mo = S.model_off
        v["slo_n"] = h["slo_n"][mo:mo + S.n_models]
        v["slo_met"] = h["slo_met"][mo:mo + S.n_models]
        v["slo_p"] = h["slo_p"][mo:mo + S.n_models]
        if "eval_report" in h:
            v["eval_report"] = h["eval_report"][s]  # [coarse, fine, adaptive][mse, p25, p50, p75, p95, n]
            v["eval_params"] = h["eval_params"][s]
            v["eval_status"] = int(h["eval_status"][s])
        return v


SEGMENTED_MIN_REQ = 2048  # request capacity from which a single-scenario batch replays as busy-period jobs


def run_batch(specs, table: _pack.TableArrays, preds=(), slo=True, warmup_fraction=0.0, arrivals=None,
              seg_stride: int = 64, max_retries: int = 4, fetch: bool = True):
    """Run a batch of scenarios to completion, growing capacities on
    overflow; returns (pipeline, fetched host dict) -- with fetch=False only
    the per-scenario counters (n_req, n_batches, n_segments, n_reseats,
    status) are copied and the results stay on the device."""
    scale = 1.0
    list_caps = None
    if arrivals is not None:
        list_caps = []
        for (tt, mm), spec in zip(arrivals, specs):
            cnt = np.bincount(np.asarray(mm, dtype=np.int64), minlength=len(spec["deployed"]))
            list_caps += [int(c) for c in cnt]
    for _ in range(max_retries + 1):
        pipe = ReplayPipeline(specs, table, seg_stride=seg_stride, scale=scale, preds=preds, list_caps=list_caps)
        wc = None
        if arrivals is not None:
            pipe.load_arrivals([a[0] for a in arrivals], [a[1] for a in arrivals])
        # one long scenario (a run_scenario call): its busy periods replay as
        # parallel jobs instead of one warp's chain (bit-identical; the bundled
        # trace's device pass 2.3 -> 0.7 ms, tools/single_trace_seg.py)
        segmented = pipe.pb.n_scen == 1 and pipe.pb.max_req_cap >= SEGMENTED_MIN_REQ

        def replay(slo_, features_):
            if segmented:
                replay_segmented(pipe, min_len=16, passes=3, arrivals=arrivals is None, slo=slo_, features=features_,
                                 stats=False)()
            else:
                pipe.run(arrivals=arrivals is None, slo=slo_, features=features_)

        if warmup_fraction:
            # cutoff = t0 + f*(t1 - t0) over the observed arrival span (`metrics.py:62-65`);
            # computed after arrivals exist (device arrays), so replay first
            replay(False, False)
            wc = _warm_cutoffs(pipe, warmup_fraction)
            pipe.run_slo_features(wc)
        else:
            replay(slo, True)
        st = pipe.status()
        if np.any(st & _abi.ST_OVERFLOW):
            scale *= 2.0
            continue
        if np.any(st & _abi.ST_SEG_STRIDE):
            seg_stride *= 4
            continue
        if not fetch:
            S = pipe.pb.n_scen
            return pipe, {k: pipe.t[k][:S].cpu().numpy() for k in ("n_req", "n_batches", "n_segments", "n_reseats",
                                                                   "status")}
        return pipe, pipe.fetch()
    raise RuntimeError("replay buffers still overflowing after retries")


def _warm_cutoffs(pipe: ReplayPipeline, frac: float):
    h_n = pipe.t["n_req"][: pipe.pb.n_scen].cpu().numpy()
    at = pipe.t["arr_t"].cpu().numpy()
    cut = np.full(pipe.pb.n_scen, -np.inf)
    for s in range(pipe.pb.n_scen):
        S = pipe.pb.scen[s]
        n = int(h_n[s])
        if n:
            seg = at[S.req_off:S.req_off + n]
            t0, t1 = float(seg.min()), float(seg.max())
            cut[s] = t0 + frac * (t1 - t0)
    return to_device(cut, pipe.dev)



# ---------------------------------------------------------------- array ops
def _f64(a, dev, shape=None):
    t = torch.from_numpy(np.array(a, dtype=np.float64, copy=True))
    if shape is not None:
        t = t.reshape(shape)
    return t.to(dev)


def _preds_struct(preds):
    n = len(preds)
    return (_abi.Predictor * max(n, 1))(*preds), n


def features_rows(own, seg_off, nseg, colo, measured, profiled, preds, want_x=True):
    """`colocation.py:95-105` over outcome rows -> (X[p][n][6], y[n], yhat[p][n]) numpy."""
    dev = require_cuda()
    n = len(seg_off)
    P, npred = _preds_struct(preds)
    d_own = _f64(own, dev)
    d_off = torch.as_tensor(np.ascontiguousarray(seg_off, dtype=np.int64)).to(dev)
    d_ns = torch.as_tensor(np.ascontiguousarray(nseg, dtype=np.int32)).to(dev)
    d_colo = _f64(colo if len(colo) else np.zeros((1, 3)), dev)
    d_m, d_p = _f64(measured, dev), _f64(profiled, dev)
    X = torch.empty(max(npred, 1) * max(n, 1) * 6, dtype=torch.float64, device=dev) if want_x else None
    y = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    yh = torch.empty(max(npred, 1) * max(n, 1), dtype=torch.float64, device=dev)
    _abi.check(_abi.load().intf_features_rows(d_own.data_ptr(), d_off.data_ptr(), d_ns.data_ptr(), d_colo.data_ptr(),
                                              d_m.data_ptr(), d_p.data_ptr(), n,
                                              ctypes.cast(P, ctypes.c_void_p) if npred else None, npred,
                                              _abi.addr(X), y.data_ptr(), yh.data_ptr(), stream_ptr()),
               "intf_features_rows")
    Xh = X.cpu().numpy()[: npred * n * 6].reshape(npred, n, 6) if want_x else None
    return Xh, y.cpu().numpy()[:n], yh.cpu().numpy()[: npred * n].reshape(npred, n)


def predict_rows(X, w7) -> np.ndarray:
    dev = require_cuda()
    X = np.asarray(X, dtype=np.float64).reshape(-1, 6)
    n = len(X)
    if n == 0:
        return np.zeros(0)
    dX, dw = _f64(X, dev), _f64(w7, dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    _abi.check(_abi.load().intf_predict_rows(dX.data_ptr(), n, dw.data_ptr(), out.data_ptr(), stream_ptr()),
               "intf_predict_rows")
    return out.cpu().numpy()


def quantiles(values, ps) -> np.ndarray:
    dev = require_cuda()
    v = _f64(values, dev)
    p = _f64(ps, dev)
    out = torch.empty(len(ps), dtype=torch.float64, device=dev)
    _abi.check(_abi.load().intf_quantiles(v.data_ptr(), v.numel(), p.data_ptr(), len(ps), out.data_ptr(), stream_ptr()),
               "intf_quantiles")
    return out.cpu().numpy()


def latency_report(group, arrival, completion, met, n_groups, cutoff=-np.inf):
    dev = require_cuda()
    g = torch.as_tensor(np.ascontiguousarray(group, dtype=np.int32)).to(dev)
    a, c = _f64(arrival, dev), _f64(completion, dev)
    m = torch.as_tensor(np.ascontiguousarray(met, dtype=np.uint8)).to(dev)
    on = torch.empty(n_groups, dtype=torch.int32, device=dev)
    om = torch.empty(n_groups, dtype=torch.int32, device=dev)
    op = torch.empty(3 * n_groups, dtype=torch.float64, device=dev)
    _abi.check(_abi.load().intf_latency_report(g.data_ptr(), a.data_ptr(), c.data_ptr(), m.data_ptr(), g.numel(),
                                               n_groups, float(cutoff), on.data_ptr(), om.data_ptr(), op.data_ptr(),
                                               stream_ptr()), "intf_latency_report")
    return on.cpu().numpy(), om.cpu().numpy(), op.cpu().numpy().reshape(n_groups, 3)


def ols_stats(X, y, out=None):
    """Z^T Z | Z^T y accumulation (`predict.py:56-63`) -> device double[56]."""
    dev = require_cuda()
    dX = X if isinstance(X, torch.Tensor) else _f64(np.asarray(X, dtype=np.float64).reshape(-1, 6), dev)
    dy = y if isinstance(y, torch.Tensor) else _f64(y, dev)
    if out is None:
        out = torch.zeros(56, dtype=torch.float64, device=dev)
    ws = torch.empty(_abi.OLS_WS_DOUBLES, dtype=torch.float64, device=dev)
    _abi.check(_abi.load().intf_ols_stats(dX.data_ptr(), dy.data_ptr(), dy.numel(), out.data_ptr(), ws.data_ptr(),
                                          stream_ptr()), "intf_ols_stats")
    return out


def ols_solve(stats, want_pinv=False):
    """-> (params[7], ridge_used, nonfinite, Pinv or None) on host."""
    dev = require_cuda()
    params = torch.empty(7, dtype=torch.float64, device=dev)
    info = torch.zeros(2, dtype=torch.int32, device=dev)
    pinv = torch.empty(49, dtype=torch.float64, device=dev) if want_pinv else None
    _abi.check(_abi.load().intf_ols_solve(stats.data_ptr(), params.data_ptr(), info.data_ptr(), _abi.addr(pinv),
                                          stream_ptr()), "intf_ols_solve")
    inf = info.cpu().numpy()
    return (params.cpu().numpy(), bool(inf[0]), bool(inf[1]),
            pinv.cpu().numpy().reshape(7, 7) if want_pinv else None)


def ols_fit(X, y):
    """fit_ols_xy on the device (`predict.py:53-66`): statistics, then the
    solve; an ill-conditioned design takes its rank (and its rank-7
    solution) from a QR of its rows.  -> (params[7], ridge_used, nonfinite)."""
    dev = require_cuda()
    dX = X if isinstance(X, torch.Tensor) else _f64(np.asarray(X, dtype=np.float64).reshape(-1, 6), dev)
    dy = y if isinstance(y, torch.Tensor) else _f64(y, dev)
    stats = ols_stats(dX, dy)
    ws = torch.empty(_abi.OLS_FIT_WS_DOUBLES, dtype=torch.float64, device=dev)
    params = torch.empty(7, dtype=torch.float64, device=dev)
    info = torch.zeros(2, dtype=torch.int32, device=dev)
    _abi.check(_abi.load().intf_ols_fit_rows(dX.data_ptr(), dy.data_ptr(), dy.numel(), stats.data_ptr(),
                                             ws.data_ptr(), params.data_ptr(), info.data_ptr(), None, stream_ptr()),
               "intf_ols_fit_rows")
    inf = info.cpu().numpy()
    return params.cpu().numpy(), bool(inf[0]), bool(inf[1])


def ols_windows(X, y, window: int):
    """fit_ols_xy on every window of `window` consecutive rows -> host
    (params[n_win, 7], info[n_win, 3]).  One launch: tensor-map staged when
    the window is a multiple of 8 rows, thread per window otherwise (two
    launches, statistics through HBM, for windows > 128 rows)."""
    dev = require_cuda()
    dX = X if isinstance(X, torch.Tensor) else _f64(np.asarray(X, dtype=np.float64).reshape(-1, 6), dev)
    dy = y if isinstance(y, torch.Tensor) else _f64(y, dev)
    n = dy.numel()
    n_win = (n + window - 1) // window
    # statistics scratch only for the two-launch path (windows > 128 rows, not a multiple of 8)
    stats = (torch.empty(max(n_win, 1) * 56, dtype=torch.float64, device=dev)
             if window > 128 and window % 8 else None)
    params = torch.empty(max(n_win, 1) * 7, dtype=torch.float64, device=dev)
    info = torch.zeros(max(n_win, 1) * 3, dtype=torch.int32, device=dev)
    _abi.check(_abi.load().intf_ols_windows(dX.data_ptr(), dy.data_ptr(), n, int(window),
                                            stats.data_ptr() if stats is not None else None, params.data_ptr(),
                                            info.data_ptr(), stream_ptr()), "intf_ols_windows")
    return params.cpu().numpy().reshape(-1, 7)[:n_win], info.cpu().numpy().reshape(-1, 3)[:n_win]


def _streams(X_list, y_list, dev):
    off = np.zeros(len(X_list) + 1, dtype=np.int64)
    for i, y in enumerate(y_list):
        off[i + 1] = off[i] + len(y)
    X = np.concatenate([np.asarray(x, dtype=np.float64).reshape(-1, 6) for x in X_list]) if off[-1] else np.zeros((1, 6))
    Y = np.concatenate([np.asarray(y, dtype=np.float64) for y in y_list]) if off[-1] else np.zeros(1)
    return off, _f64(X, dev), _f64(Y, dev), torch.as_tensor(off).to(dev)


def sgd_streams(X_list, y_list, params, eta):
    """Prequential SGD (`predict.py:88-95,157-172`) over independent streams.
    params: [S][7] initial (w, b); eta: [S].  -> (preds list, params, status)."""
    dev = require_cuda()
    off, dX, dY, doff = _streams(X_list, y_list, dev)
    S = len(X_list)
    dp = _f64(params, dev)
    de = _f64(np.broadcast_to(np.asarray(eta, dtype=np.float64), (S,)), dev)
    pred = torch.empty(max(int(off[-1]), 1), dtype=torch.float64, device=dev)
    st = torch.zeros(max(S, 1), dtype=torch.int32, device=dev)
    _abi.check(_abi.load().intf_sgd_streams(dX.data_ptr(), dY.data_ptr(), doff.data_ptr(), S, de.data_ptr(),
                                            dp.data_ptr(), pred.data_ptr(), st.data_ptr(), stream_ptr()),
               "intf_sgd_streams")
    ph = pred.cpu().numpy()
    return [ph[off[i]:off[i + 1]] for i in range(S)], dp.cpu().numpy().reshape(S, 7), st.cpu().numpy()[:S]


def rls_streams(X_list, y_list, params, P, lam):
    """Prequential RLS (`predict.py:137-154,157-172`).  -> (preds, params, P, status)."""
    dev = require_cuda()
    off, dX, dY, doff = _streams(X_list, y_list, dev)
    S = len(X_list)
    dp = _f64(params, dev)
    dP = _f64(P, dev)
    dl = _f64(np.broadcast_to(np.asarray(lam, dtype=np.float64), (S,)), dev)
    pred = torch.empty(max(int(off[-1]), 1), dtype=torch.float64, device=dev)
    st = torch.zeros(max(S, 1), dtype=torch.int32, device=dev)
    _abi.check(_abi.load().intf_rls_streams(dX.data_ptr(), dY.data_ptr(), doff.data_ptr(), S, dl.data_ptr(),
                                            dp.data_ptr(), dP.data_ptr(), pred.data_ptr(), st.data_ptr(), stream_ptr()),
               "intf_rls_streams")
    ph = pred.cpu().numpy()
    return ([ph[off[i]:off[i + 1]] for i in range(S)], dp.cpu().numpy().reshape(S, 7),
            dP.cpu().numpy().reshape(S, 7, 7), st.cpu().numpy()[:S])


def eval_reports(yhat_list, y_list) -> np.ndarray:
    """EvalReport rows (`predict.py:195-205`): [S][6] = mse, p25, p50, p75, p95, n."""
    dev = require_cuda()
    off = np.zeros(len(y_list) + 1, dtype=np.int64)
    for i, y in enumerate(y_list):
        off[i + 1] = off[i] + len(y)
    yh = _f64(np.concatenate([np.asarray(a, dtype=np.float64) for a in yhat_list]), dev)
    yy = _f64(np.concatenate([np.asarray(a, dtype=np.float64) for a in y_list]), dev)
    doff = torch.as_tensor(off).to(dev)
    out = torch.empty(6 * len(y_list), dtype=torch.float64, device=dev)
    _abi.check(_abi.load().intf_eval_report(yh.data_ptr(), yy.data_ptr(), doff.data_ptr(), len(y_list), out.data_ptr(),
                                            stream_ptr()), "intf_eval_report")
    return out.cpu().numpy().reshape(-1, 6)


def candidate_layout(n_rows: int, cap: int) -> tuple:
    """(n_cand, n_sets, ld) of the candidate enumeration (intf_candidate_count)."""
    n, s, ld = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    _abi.check(_abi.load().intf_candidate_count(n_rows, cap, ctypes.byref(n), ctypes.byref(s), ctypes.byref(ld)),
               "intf_candidate_count")
    return int(n.value), int(s.value), int(ld.value)


def candidate_count(n_rows: int, cap: int) -> int:
    return candidate_layout(n_rows, cap)[0]


class CandidateScorer:
    """Every candidate co-location set over a profile table,
    scored by a coarse (static) and a fine (EWMA) linear predictor for n_dec
    decisions.  Output (device, fp32) in the tiled HBM layout of the kernels
    (csrc/predict.cu): tiles [ceil(n_dec/4)][E][ld/512] of [4 dec][2 kinds]
    [512 multisets]; `view` returns the logical [n_dec][2][E][n_sets] array
    (ld = n_sets rounded up to 512, pad lanes written as 0)."""

    TILE_R, TILE_D = 512, 4

    def __init__(self, table: _pack.TableArrays, cap: int, alpha: float = 0.5, dtable: DeviceTable | None = None,
                 two_phase: bool = True):
        self.dev = require_cuda()
        self.dtable = dtable or DeviceTable(table, self.dev)
        self.E = table.n_rows
        self.cap = int(cap)
        self.alpha = float(alpha)
        self.n_cand, self.n_sets, self.ld = candidate_layout(self.E, self.cap)
        ws = ctypes.c_int64(0)
        _abi.check(_abi.load().intf_candidate_workspace(self.E, self.cap, ctypes.byref(ws)), "intf_candidate_workspace")
        self.ws_elems = int(ws.value) if two_phase else 0
        self.ws = torch.empty(max(self.ws_elems, 1), dtype=torch.float32, device=self.dev) if two_phase else None

    def out_elems(self, n_dec: int) -> int:
        return -(-n_dec // self.TILE_D) * self.TILE_D * 2 * self.E * self.ld

    def alloc(self, n_dec: int) -> torch.Tensor:
        return torch.empty(self.out_elems(n_dec), dtype=torch.float32, device=self.dev)

    def view(self, out, n_dec: int):
        """[n_dec, 2, E, n_sets] view of an output buffer (torch or numpy)."""
        return self.view_full(out, n_dec)[..., : self.n_sets]

    def view_full(self, out, n_dec: int):
        """[n_dec, 2, E, ld] logical array (incl. pad lanes) of an output
        buffer in the tiled layout (a copy; numpy or torch)."""
        dc, rc, T = -(-n_dec // self.TILE_D), self.ld // self.TILE_R, self.TILE_R
        t = out.reshape(dc, self.E, rc, self.TILE_D, 2, T)
        t = t.permute(0, 3, 4, 1, 2, 5) if hasattr(t, "permute") else t.transpose(0, 3, 4, 1, 2, 5)
        return t.reshape(dc * self.TILE_D, 2, self.E, rc * T)[:n_dec]

    def score(self, coefs: torch.Tensor, out: torch.Tensor) -> None:
        """coefs: device float64 [n_dec][2][7]; enqueue only (no sync)."""
        n_dec = coefs.numel() // 14
        _abi.check(_abi.load().intf_predict_candidates(ctypes.byref(self.dtable.struct), self.cap, self.alpha,
                                                       coefs.data_ptr(), n_dec, out.data_ptr(), _abi.addr(self.ws),
                                                       self.ws_elems, stream_ptr()), "intf_predict_candidates")

    def prepare(self) -> None:
        """Phase 1 only (k_cand_prep): candidate features into the workspace."""
        _abi.check(_abi.load().intf_candidate_prepare(ctypes.byref(self.dtable.struct), self.cap, self.alpha,
                                                      _abi.addr(self.ws), self.ws_elems, stream_ptr()),
                   "intf_candidate_prepare")

    def score_prepared(self, coefs: torch.Tensor, out: torch.Tensor) -> None:
        """Phase 2 only (k_cand_stream) from a prepared workspace."""
        n_dec = coefs.numel() // 14
        _abi.check(_abi.load().intf_predict_candidates_prepared(ctypes.byref(self.dtable.struct), self.cap,
                                                                coefs.data_ptr(), n_dec, out.data_ptr(),
                                                                _abi.addr(self.ws), self.ws_elems, stream_ptr()),
                   "intf_predict_candidates_prepared")

    def pipeline_start(self, fused: bool = True) -> None:
        """Start a pipelined sequence of steps (`pipeline_step`): features for
        the first step are built now (k_cand_prep) into workspace 0.
        fused: each step is ONE k_cand_step launch (forward of this step +
        feature build of the next, horizontally fused); otherwise the feature
        build runs as k_cand_prep on a side stream beside k_cand_stream."""
        s = torch.cuda.current_stream(self.dev)
        if getattr(self, "_ws", None) is None:
            self._side = torch.cuda.Stream(self.dev)
            self._ws = [self.ws, torch.empty_like(self.ws)]
            self._ready = [torch.cuda.Event(), torch.cuda.Event()]
            self._read = [torch.cuda.Event(), torch.cuda.Event()]
        self._k = 0
        self._fused = bool(fused)
        self._prepare_into(self._ws[0], s)
        self._ready[0].record(s)

    def _prepare_into(self, ws: torch.Tensor, s: torch.cuda.Stream) -> None:
        _abi.check(_abi.load().intf_candidate_prepare(ctypes.byref(self.dtable.struct), self.cap, self.alpha,
                                                      ws.data_ptr(), self.ws_elems, s.cuda_stream),
                   "intf_candidate_prepare")

    def pipeline_step(self, coefs: torch.Tensor, out: torch.Tensor, kernel_events=None) -> None:
        """One step = the forward of every candidate for coefs' decisions,
        from the features built for this step, + the feature build for the
        NEXT step into the other workspace.  The forward is HBM-write bound
        and the feature build issue/L2 bound, so the two overlap.
        kernel_events = (start, end) CUDA events bracketing the forward launch."""
        s = torch.cuda.current_stream(self.dev)
        cur, nxt = self._k & 1, (self._k + 1) & 1
        n_dec = coefs.numel() // 14
        L = _abi.load()
        if self._fused:
            if kernel_events:
                kernel_events[0].record(s)
            _abi.check(L.intf_candidate_step(ctypes.byref(self.dtable.struct), self.cap, self.alpha,
                                             coefs.data_ptr(), n_dec, out.data_ptr(), self._ws[cur].data_ptr(),
                                             self._ws[nxt].data_ptr(), self.ws_elems, s.cuda_stream),
                       "intf_candidate_step")
            if kernel_events:
                kernel_events[1].record(s)
            self._k += 1
            return
        s.wait_event(self._ready[cur])
        if kernel_events:
            kernel_events[0].record(s)
        _abi.check(L.intf_predict_candidates_prepared(ctypes.byref(self.dtable.struct), self.cap, coefs.data_ptr(),
                                                      n_dec, out.data_ptr(), self._ws[cur].data_ptr(), self.ws_elems,
                                                      s.cuda_stream), "intf_predict_candidates_prepared")
        if kernel_events:
            kernel_events[1].record(s)
        self._read[cur].record(s)
        # next step's features: after the previous step's forward released that workspace
        side = self._side
        side.wait_event(self._read[nxt]) if self._k > 0 else side.wait_stream(s)
        self._prepare_into(self._ws[nxt], side)
        self._ready[nxt].record(side)
        self._k += 1

    # ---- best candidate per (decision, kind, own): the reduction a scheduler consumes
    def alloc_best(self, n_dec: int) -> torch.Tensor:
        """Key buffer [n_dec][2][E] (int64 view of the u64 keys), reset to the all-ones key."""
        return torch.full((2 * n_dec * self.E,), -1, dtype=torch.int64, device=self.dev)

    def best_step(self, coefs: torch.Tensor, best: torch.Tensor, best_next: torch.Tensor, kernel_events=None) -> None:
        """One pipelined step (after pipeline_start(fused=True)) that scores
        every candidate of coefs' decisions but keeps only the best one per
        (decision, kind, own) in `best` (intf_candidate_best_step); resets
        best_next and builds the next step's features in the same launch."""
        s = torch.cuda.current_stream(self.dev)
        cur, nxt = self._k & 1, (self._k + 1) & 1
        if kernel_events:
            kernel_events[0].record(s)
        _abi.check(_abi.load().intf_candidate_best_step(ctypes.byref(self.dtable.struct), self.cap, self.alpha,
                                                        coefs.data_ptr(), coefs.numel() // 14, best.data_ptr(),
                                                        best_next.data_ptr(), self._ws[cur].data_ptr(),
                                                        self._ws[nxt].data_ptr(), self.ws_elems, s.cuda_stream),
                   "intf_candidate_best_step")
        if kernel_events:
            kernel_events[1].record(s)
        self._k += 1

    def best_scratch_elems(self, n_dec: int) -> int:
        """Device floats needed by best_host."""
        return 28 * n_dec + 4 * n_dec * self.E + self.ws_elems

    def best_host(self, coefs_host: np.ndarray, best_host: np.ndarray, scratch: torch.Tensor) -> None:
        """End to end, host buffers (intf_best_candidates_host): host coefs in,
        the best candidate keys [n_dec][2][E] (uint64) out; enqueue only."""
        n_dec = coefs_host.size // 14
        _abi.check(_abi.load().intf_best_candidates_host(ctypes.byref(self.dtable.struct), self.cap, self.alpha,
                                                         coefs_host.ctypes.data, n_dec, best_host.ctypes.data,
                                                         scratch.data_ptr(), scratch.numel(), stream_ptr()),
                   "intf_best_candidates_host")

    def best_host_pipelined(self, coefs_host: np.ndarray, best_host: np.ndarray, scratch: torch.Tensor,
                            sync: bool = False) -> None:
        """best_host as a pipeline of decisions (intf_best_candidates_host_pipelined):
        each call scores from the features the previous call built and builds
        the next call's in the same launch; scratch holds
        best_scratch_elems(n_dec) + one more workspace.  With a pinned
        best_host and <= 32 decisions a call is one kernel launch.  sync:
        return with the keys in best_host (intf_best_candidates_host_sync)."""
        n_dec = coefs_host.size // 14
        c = getattr(self, "_host_call", None)
        if c is None:  # per-call marshalling cached (a call is ~50 us; the argument objects cost ~5)
            self._host_state = np.zeros(1, dtype=np.int64)
            L = _abi.load()
            c = self._host_call = {"fn": L.intf_best_candidates_host_pipelined,
                                   "fn_sync": L.intf_best_candidates_host_sync,
                                   "table": ctypes.byref(self.dtable.struct),
                                   "state": self._host_state.ctypes.data, "ptrs": {}}
        ptrs = c["ptrs"]

        def ptr(a):
            hit = ptrs.get(id(a))
            if hit is None or hit[0] is not a:
                if len(ptrs) > 64:
                    ptrs.clear()
                hit = ptrs[id(a)] = (a, a.ctypes.data)
            return hit[1]

        _abi.check(c["fn_sync" if sync else "fn"](c["table"], self.cap, self.alpha, ptr(coefs_host), n_dec,
                                                   ptr(best_host), scratch.data_ptr(), scratch.numel(), c["state"],
                                                   torch.cuda.current_stream().cuda_stream),
                   "intf_best_candidates_host_sync" if sync else "intf_best_candidates_host_pipelined")

    def decode_best(self, keys, n_dec: int):
        """(value [n_dec][2][E] float32, multiset rank [n_dec][2][E] int64) of
        best keys (torch or numpy, int64 or uint64)."""
        k = np.asarray(keys.cpu().numpy() if hasattr(keys, "cpu") else keys).view(np.uint64).reshape(n_dec, 2, self.E)
        hi = (k >> np.uint64(32)).astype(np.uint32)
        bits = np.where(hi >> np.uint32(31), hi & np.uint32(0x7FFFFFFF), ~hi).astype(np.uint32)
        return bits.view(np.float32), (k & np.uint64(0xFFFFFFFF)).astype(np.int64)

    # ---- real decisions: the running set at every dispatch of a replayed batch
    def dispatch_decisions(self, pipe: "ReplayPipeline"):
        """(dec_rank, dec_own) per batch slot of a replayed pipeline
        (intf_dispatch_sets): the running set at each dispatch as a column of
        this scorer's enumeration, and the dispatched batch's own row."""
        n = int(pipe.batch.req_slots)
        rank = torch.empty(n, dtype=torch.int32, device=self.dev)
        own = torch.empty(n, dtype=torch.int32, device=self.dev)
        _abi.check(_abi.load().intf_dispatch_sets(ctypes.byref(pipe.batch), ctypes.byref(pipe.B), self.E, self.cap,
                                                  rank.data_ptr(), own.data_ptr(), stream_ptr()),
                   "intf_dispatch_sets")
        return rank, own

    def score_decisions(self, coefs: torch.Tensor, rank: torch.Tensor, own: torch.Tensor, best=None, chosen=None):
        """Every own row against each decision's running set under one coarse /
        fine model coefs[2][7] (device f64; features from prepare()):
        best keys [n][2] (int64 view of u64) and the FIFO batch's predictions
        [n][2]; enqueue only."""
        n = rank.numel()
        best = best if best is not None else torch.empty(2 * n, dtype=torch.int64, device=self.dev)
        chosen = chosen if chosen is not None else torch.empty(2 * n, dtype=torch.float32, device=self.dev)
        ft = getattr(self, "_ft", None)
        _abi.check(_abi.load().intf_score_decisions_ft(ctypes.byref(self.dtable.struct), self.cap, coefs.data_ptr(),
                                                       self.ws.data_ptr(), self.ws_elems, _abi.addr(ft),
                                                       rank.data_ptr(), own.data_ptr(), n, best.data_ptr(),
                                                       chosen.data_ptr(), stream_ptr()), "intf_score_decisions_ft")
        return best, chosen

    def prepare_decisions(self) -> None:
        """prepare() + the decision-major copy of the EWMA features
        (intf_decision_features) used by score_decisions."""
        L = _abi.load()
        self.prepare()
        n = int(L.intf_decision_features_elems(self.E, self.cap))
        if getattr(self, "_ft", None) is None or self._ft.numel() != n:
            self._ft = torch.empty(n, dtype=torch.float32, device=self.dev)
        _abi.check(L.intf_decision_features(ctypes.byref(self.dtable.struct), self.cap, self.ws.data_ptr(),
                                            self.ws_elems, self._ft.data_ptr(), stream_ptr()), "intf_decision_features")

    def pipeline_join(self) -> None:
        """Make the current stream wait for the side stream's last feature build."""
        if not self._fused:
            torch.cuda.current_stream(self.dev).wait_stream(self._side)

    def scratch_elems(self, n_dec: int) -> int:
        """Device floats needed by score_host (coefs + outputs + workspace)."""
        return 28 * n_dec + self.out_elems(n_dec) + self.ws_elems

    def score_host(self, coefs_host: np.ndarray, out_host: np.ndarray, scratch: torch.Tensor) -> None:
        """End-to-end variant: host coefs in, host predictions out."""
        n_dec = coefs_host.size // 14
        _abi.check(_abi.load().intf_predict_candidates_host(ctypes.byref(self.dtable.struct), self.cap, self.alpha,
                                                            coefs_host.ctypes.data, n_dec, out_host.ctypes.data,
                                                            scratch.data_ptr(), scratch.numel(), stream_ptr()),
                   "intf_predict_candidates_host")


def multiset_rank(peers, E: int, cap: int) -> int:
    """Index of a peer multiset within one own row (size-major, colex)."""
    p = sorted(int(q) for q in peers)
    k = len(p)
    r = sum(_comb(E + j - 1, j) for j in range(k))
    for i, q in enumerate(p, start=1):
        r += _comb(q + i - 1, i)
    return r


def _comb(n: int, k: int) -> int:
    import math

    return math.comb(n, k) if 0 <= k <= n else 0


def arrivals(specs, table: _pack.TableArrays, max_retries: int = 6):
    """generate_arrivals for a batch of scenario dicts (`workload.py:74-104`)
    -> list of (arrival_ms, deployed index) numpy pairs."""
    scale = 1.0
    for _ in range(max_retries + 1):
        pipe = ReplayPipeline(specs, table, scale=scale, seg_stride=1)
        _abi.check(_abi.load().intf_generate_arrivals(ctypes.byref(pipe.batch), ctypes.byref(pipe.B), stream_ptr()),
                   "intf_generate_arrivals")
        if np.any(pipe.status() & _abi.ST_OVERFLOW):
            scale *= 2.0
            continue
        n_req = pipe.t["n_req"][: pipe.pb.n_scen].cpu().numpy()
        at, am = pipe.t["arr_t"].cpu().numpy(), pipe.t["arr_model"].cpu().numpy()
        out = []
        for s in range(pipe.pb.n_scen):
            S = pipe.pb.scen[s]
            out.append((at[S.req_off:S.req_off + n_req[s]].copy(), am[S.req_off:S.req_off + n_req[s]].copy()))
        return out
    raise RuntimeError("arrival buffers still overflowing after retries")


SCALAR_NOISE, SCALAR_SLOWDOWN, SCALAR_PREDICT, SCALAR_EWMA, SCALAR_SGD, SCALAR_RLS = range(6)
_SCALAR_OUT = {SCALAR_NOISE: 1, SCALAR_SLOWDOWN: 1, SCALAR_PREDICT: 1, SCALAR_EWMA: 3, SCALAR_SGD: 9, SCALAR_RLS: 58}


def scalar(op: int, ints=(), floats=()) -> np.ndarray:
    """One scalar call (intf_scalar): `ints` as uint64 words, then `floats`
    by their float64 bits; returns the op's outputs (float64)."""
    require_cuda()
    args = np.concatenate([np.asarray(ints, dtype=np.uint64).reshape(-1),
                           np.ascontiguousarray(np.asarray(floats, dtype=np.float64).reshape(-1)).view(np.uint64)])
    n_out = _SCALAR_OUT[op]
    out = np.empty(n_out, dtype=np.float64)
    _abi.check(_abi.load().intf_scalar(op, args.ctypes.data, len(args), out.ctypes.data, n_out, stream_ptr()),
               "intf_scalar")
    return out


def noise_draws(seed: int, sigma: float, batch_ids, seg_idx) -> np.ndarray:
    dev = require_cuda()
    b = torch.as_tensor(np.ascontiguousarray(batch_ids, dtype=np.int64)).to(dev)
    k = torch.as_tensor(np.ascontiguousarray(seg_idx, dtype=np.int64)).to(dev)
    out = torch.empty(max(b.numel(), 1), dtype=torch.float64, device=dev)
    _abi.check(_abi.load().intf_noise_draws(int(seed), float(sigma), b.data_ptr(), k.data_ptr(), b.numel(),
                                            out.data_ptr(), stream_ptr()), "intf_noise_draws")
    return out.cpu().numpy()[: b.numel()]


def slowdowns(own, colo, beta, noise=None) -> np.ndarray:
    dev = require_cuda()
    o, c = _f64(np.asarray(own).reshape(-1, 3), dev), _f64(np.asarray(colo).reshape(-1, 3), dev)
    bt = np.ascontiguousarray(beta, dtype=np.float64)  # host array (read at launch)
    nz = _f64(noise, dev) if noise is not None else None
    n = o.shape[0]
    out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    _abi.check(_abi.load().intf_slowdowns(o.data_ptr(), c.data_ptr(), bt.ctypes.data, _abi.addr(nz), n, out.data_ptr(),
                                          stream_ptr()), "intf_slowdowns")
    return out.cpu().numpy()[:n]


def rng_stream(words, n: int, uniform: bool = False) -> np.ndarray:
    dev = require_cuda()
    w = torch.as_tensor(np.ascontiguousarray(words, dtype=np.uint32).view(np.int32)).to(dev)
    out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    _abi.check(_abi.load().intf_rng_stream(w.data_ptr(), w.numel(), n, int(uniform), out.data_ptr(), stream_ptr()),
               "intf_rng_stream")
    return out.cpu().numpy()[:n]


# ------------------------------------------------------ busy-period sharding
def _candidate_starts(pipe, nb, formed_all, bmod, bsz, slow: float, min_len: int):
    """Speculative job starts for every scenario (vectorised): batch b starts
    a job if it forms after every earlier batch's optimistic end
    formed + slow * solo (running max within its scenario) and the job before
    it has at least min_len batches.  Only a speculation -- the replay
    verifies each boundary exactly.  Returns (scen, lo) arrays, sorted."""
    S_n = pipe.pb.n_scen
    req_off = np.array([pipe.pb.scen[s].req_off for s in range(S_n)], dtype=np.int64)
    nbv = nb.astype(np.int64)
    tot = int(nbv.sum())
    if tot == 0:
        return np.arange(S_n, dtype=np.int32), np.zeros(S_n, dtype=np.int32)
    scen = np.repeat(np.arange(S_n), nbv)
    local = np.arange(tot) - np.repeat(np.cumsum(nbv) - nbv, nbv)
    slot = req_off[scen] + local
    mbase = np.array([pipe.pb.models[g].entry_base for g in range(max(pipe.pb.n_models, 1))], dtype=np.int64)
    moff = np.array([pipe.pb.scen[s].model_off for s in range(S_n)], dtype=np.int64)
    rows = mbase[moff[scen] + bmod[slot]] + bsz[slot] - 1
    f = formed_all[slot]
    end = f + slow * pipe.pb.table.solo[rows]
    # running max of `end` restricted to each scenario: offset scenarios apart
    big = (np.abs(end).max() + np.abs(f).max() + 1.0) * 4.0
    cm = np.maximum.accumulate(end + scen * big) - scen * big
    cand = np.zeros(tot, dtype=bool)
    cand[1:] = (f[1:] > cm[:-1]) & (scen[1:] == scen[:-1])
    first = local == 0
    starts = first | cand
    idx = np.nonzero(starts)[0]
    if min_len > 1 and len(idx) > 1:
        # thin to at most one candidate per min_len-batch bucket of a scenario (scenario starts always kept)
        bucket = scen[idx].astype(np.int64) * (1 << 32) + local[idx] // min_len
        first_in_bucket = np.ones(len(idx), dtype=bool)
        first_in_bucket[1:] = bucket[1:] != bucket[:-1]
        idx = idx[first_in_bucket | (local[idx] == 0)]
    js, jl = scen[idx].astype(np.int32), local[idx].astype(np.int32)
    # scenarios without batches still get one (empty) job
    empty = np.nonzero(nbv == 0)[0]
    if len(empty):
        js = np.concatenate([js, empty.astype(np.int32)])
        jl = np.concatenate([jl, np.zeros(len(empty), dtype=np.int32)])
        o = np.lexsort((jl, js))
        js, jl = js[o], jl[o]
    return js, jl


def replay_segmented_host(pipe: "ReplayPipeline", slow: float = 2.0, min_len: int = 96, max_iters: int = 100000,
                          arrivals: bool = True, slo: bool = True, features: bool = True) -> dict:
    """Busy-period sharding: replay every scenario as parallel
    jobs split at speculated idle points, verify every boundary (previous
    job's last completion <= next job's first formation), remove the failing
    ones and replay the merged jobs again until all boundaries hold.  The
    result is identical to the serial replay.  Returns statistics."""
    import time

    L, st = pipe.lib, stream_ptr()
    bt, B = ctypes.byref(pipe.batch), ctypes.byref(pipe.B)
    tm = {}
    t0 = time.perf_counter()
    if arrivals:
        _abi.check(L.intf_generate_arrivals(bt, B, st), "intf_generate_arrivals")
    else:
        _abi.check(L.intf_split_arrivals(bt, B, st), "intf_split_arrivals")
    _abi.check(L.intf_form_batches(bt, B, st), "intf_form_batches")
    nb = pipe.t["n_batches"][: pipe.pb.n_scen].cpu().numpy()
    tm["arrivals+formation"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    formed_all = pipe.t["b_formed"].cpu().numpy()
    bmod = pipe.t["b_model"].cpu().numpy()
    bsz = pipe.t["b_size"].cpu().numpy()
    js, jl = _candidate_starts(pipe, nb, formed_all, bmod, bsz, slow, min_len)
    req_off = np.array([pipe.pb.scen[s].req_off for s in range(pipe.pb.n_scen)], dtype=np.int64)

    def ends(js, jl):
        nxt_same = np.zeros(len(js), dtype=bool)
        nxt_same[:-1] = js[1:] == js[:-1]
        jh = np.where(nxt_same, np.roll(jl, -1), nb[js]).astype(np.int32)
        return jh

    jh = ends(js, jl)
    n_initial = len(js)
    tm["plan"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    need = max(n_initial, pipe.pb.n_scen) * pipe.pb.cap_max * pipe.seg_stride * 5
    if pipe.t["slot_seg"].numel() < need:
        pipe.t["slot_seg"] = torch.zeros(need, dtype=torch.float64, device=pipe.dev)
        pipe.B.slot_seg = pipe.t["slot_seg"].data_ptr()
    last = np.full(len(js), -np.inf)
    info = np.zeros((len(js), 3), dtype=np.int32)
    dirty = np.ones(len(js), dtype=bool)
    iters = 0
    for iters in range(1, max_iters + 1):
        todo = np.nonzero(dirty & (jh > jl))[0]
        if len(todo):
            d_sc = torch.from_numpy(js[todo].copy()).to(pipe.dev)
            d_lo = torch.from_numpy(jl[todo].copy()).to(pipe.dev)
            d_hi = torch.from_numpy(jh[todo].copy()).to(pipe.dev)
            d_last = torch.empty(len(todo), dtype=torch.float64, device=pipe.dev)
            d_info = torch.empty(3 * len(todo), dtype=torch.int32, device=pipe.dev)
            _abi.check(L.intf_replay_jobs(bt, ctypes.byref(pipe.dtable.struct), B, d_sc.data_ptr(), d_lo.data_ptr(),
                                          d_hi.data_ptr(), len(todo), d_last.data_ptr(), d_info.data_ptr(), st),
                       "intf_replay_jobs")
            last[todo] = d_last.cpu().numpy()
            info[todo] = d_info.cpu().numpy().reshape(-1, 3)
        dirty[:] = False
        # verify: boundary i (same scenario as i-1) holds iff last[i-1] <= formed(first batch of i)
        same = np.zeros(len(js), dtype=bool)
        same[1:] = js[1:] == js[:-1]
        prev_last = np.concatenate([[-np.inf], last[:-1]])
        ok = ~same | (jh <= jl) | (prev_last <= formed_all[req_off[js] + jl])
        if ok.all():
            break
        # drop failing boundaries; jobs that absorbed one are replayed again
        keep = ok
        grp = np.cumsum(keep) - 1
        absorbed = np.zeros(int(keep.sum()), dtype=bool)
        np.logical_or.at(absorbed, grp[~keep], True)
        js, jl = js[keep], jl[keep]
        jh = ends(js, jl)
        last, info = last[keep], info[keep]
        dirty = absorbed
    torch.cuda.synchronize()
    tm["replay+verify"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    # per-scenario totals of the final jobs
    S_n = pipe.pb.n_scen
    live = jh > jl
    status = pipe.t["status"][:S_n].cpu().numpy().copy()
    np.bitwise_or.at(status, js[live], info[live, 0])
    n_seg = np.bincount(js[live], weights=info[live, 1], minlength=S_n).astype(np.int32)
    n_res = np.bincount(js[live], weights=info[live, 2], minlength=S_n).astype(np.int32)
    pipe.t["n_segments"][:S_n].copy_(torch.from_numpy(n_seg))
    pipe.t["n_reseats"][:S_n].copy_(torch.from_numpy(n_res))
    pipe.t["status"][:S_n].copy_(torch.from_numpy(status))
    pipe.run_slo_features(slo=slo, features=features)
    torch.cuda.synchronize()
    tm["slo+features"] = time.perf_counter() - t0
    return {"jobs_initial": n_initial, "jobs_final": int(len(js)), "iterations": iters, "batches": int(nb.sum()),
            "host_wall_ms": {k: round(v * 1e3, 3) for k, v in tm.items()}}


class _DeviceJobs:
    """Job-slot buffers of the device-planned busy-period sharding."""

    def __init__(self, pipe: "ReplayPipeline", slow: float, min_len: int):
        pb = pipe.pb
        jcap = np.array([pb.scen[s].req_cap // min_len + 2 for s in range(pb.n_scen)], dtype=np.int32)
        joff = np.concatenate([[0], np.cumsum(jcap)[:-1]]).astype(np.int32)
        total = int(jcap.sum())
        dev = pipe.dev
        self.t = {
            "joff": torch.from_numpy(joff).to(dev), "jcap": torch.from_numpy(jcap).to(dev),
            "lo": torch.zeros(total, dtype=torch.int32, device=dev), "hi": torch.zeros(total, dtype=torch.int32, device=dev),
            "n_jobs": torch.zeros(pb.n_scen, dtype=torch.int32, device=dev),
            "last": torch.zeros(total, dtype=torch.float64, device=dev),
            "info": torch.zeros(3 * total, dtype=torch.int32, device=dev),
            "dirty": torch.zeros(total, dtype=torch.uint8, device=dev),
            "todo": torch.zeros(total, dtype=torch.int32, device=dev),
            "todo_count": torch.zeros(2, dtype=torch.int32, device=dev),
            "slot_scen": torch.from_numpy(np.repeat(np.arange(pb.n_scen, dtype=np.int32), jcap)).to(dev),
            "scratch": torch.zeros(6 * total, dtype=torch.float64, device=dev),  # long-trace plan/verify
        }
        self.J = _abi.Jobs(**{k: v.data_ptr() for k, v in self.t.items()}, slow=float(slow), min_len=int(min_len),
                           total_slots=total, own_lo=0, own_hi=2**31 - 1)
        self.key = (float(slow), int(min_len))


def replay_segmented(pipe: "ReplayPipeline", slow: float = 2.0, min_len: int = 96, max_iters: int = 100000,
                     arrivals: bool = True, slo: bool = True, features: bool = True, passes: int = 0,
                     stats: bool = True) -> dict:
    """Busy-period sharding, planned and verified on the device:
    speculative idle boundaries (k_jobs_plan), parallel job replay
    (k_jobs_replay), boundary verification and merging (k_jobs_verify),
    repeated until every boundary holds.  Bit-identical to the serial replay.
    passes > 0: that many replay + verify passes are queued with the job
    count read ON THE DEVICE (no host round trip; spare passes find an empty
    todo list), then the host checks the count once and continues if needed.
    passes = 0: the host reads the todo-list size between launches.
    stats=False skips the statistics' host reads (nothing left to sync on:
    the whole call is stream-ordered)."""
    L, st = pipe.lib, stream_ptr()
    bt, B = ctypes.byref(pipe.batch), ctypes.byref(pipe.B)
    jobs = getattr(pipe, "_jobs", None)
    if jobs is None or jobs.key != (float(slow), int(min_len)):
        jobs = _DeviceJobs(pipe, slow, min_len)
        pipe._jobs = jobs
    J = ctypes.byref(jobs.J)
    if arrivals:
        _abi.check(L.intf_generate_arrivals(bt, B, st), "intf_generate_arrivals")
    else:
        _abi.check(L.intf_split_arrivals(bt, B, st), "intf_split_arrivals")
    _abi.check(L.intf_form_batches(bt, B, st), "intf_form_batches")
    tab = ctypes.byref(pipe.dtable.struct)
    _abi.check(L.intf_jobs_plan(bt, tab, B, J, st), "intf_jobs_plan")
    iters, first = 0, None
    if passes > 0:
        total = int(jobs.J.total_slots)
        need = total * pipe.pb.cap_max * pipe.seg_stride * 5
        if pipe.t["slot_seg"].numel() < need:
            pipe.t["slot_seg"] = torch.zeros(need, dtype=torch.float64, device=pipe.dev)
            pipe.B.slot_seg = pipe.t["slot_seg"].data_ptr()
        if stats:
            jobs.t["n_jobs0"] = jobs.t["n_jobs"].clone()
        for _ in range(passes):
            _abi.check(L.intf_jobs_replay(bt, tab, B, J, -total, st), "intf_jobs_replay")
            _abi.check(L.intf_jobs_verify(bt, B, J, st), "intf_jobs_verify")
        iters = passes
        if not stats:
            # deferred: SLO / features queued now; finish() (one host read)
            # checks that the passes sufficed, else completes and redoes them
            pipe.run_slo_features(slo=slo, features=features)

            def finish() -> dict:
                if int(jobs.t["todo_count"][0].item()) == 0:
                    return {"iterations": passes}
                return replay_segmented_continue(pipe, jobs, passes, max_iters, slo, features, None)

            return finish
        first = int(jobs.t["n_jobs0"].sum().item())
    return replay_segmented_continue(pipe, jobs, iters, max_iters, slo, features, first)


def replay_segmented_continue(pipe, jobs, iters, max_iters, slo, features, first) -> dict:
    """The host-driven tail of replay_segmented: read the todo-list size,
    replay and verify until it is empty, then SLO / features."""
    L, st = pipe.lib, stream_ptr()
    bt, B, J = ctypes.byref(pipe.batch), ctypes.byref(pipe.B), ctypes.byref(jobs.J)
    tab = ctypes.byref(pipe.dtable.struct)
    for iters in range(iters + 1, max_iters + 1):
        n = int(jobs.t["todo_count"][0].item())
        if first is None:
            first = n
        if n == 0:
            break
        need = n * pipe.pb.cap_max * pipe.seg_stride * 5
        if pipe.t["slot_seg"].numel() < need:
            pipe.t["slot_seg"] = torch.zeros(need, dtype=torch.float64, device=pipe.dev)
            pipe.B.slot_seg = pipe.t["slot_seg"].data_ptr()
        _abi.check(L.intf_jobs_replay(bt, tab, B, J, n, st), "intf_jobs_replay")
        _abi.check(L.intf_jobs_verify(bt, B, J, st), "intf_jobs_verify")
    pipe.run_slo_features(slo=slo, features=features)
    final = int(jobs.t["n_jobs"].sum().item())
    return {"jobs_initial": int(first or 0), "jobs_final": final, "iterations": iters,
            "batches": int(pipe.t["n_batches"][: pipe.pb.n_scen].sum().item())}
