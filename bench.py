"""Benchmark of the intfsim hot path on B200 (contract: one JSON line).

Headline workload (BASELINE.json configs[1], C2): every candidate co-located
batch set over the 48 bundled profile entries at concurrency cap 4 (999,600
own x peer-multiset candidates), scored by the coarse (static
features) and fine (EWMA(1/2) features) linear predictors for D = 32
scheduling decisions per step, each decision with its own refit
coefficients (OLS on growing windows of the bundled trace's samples).
One step = one k_cand_step launch: its stream blocks write 63,974,400 fp32
predictions (256 MB > L2, so no flush is needed between steps) and its prep
blocks build the candidate features for the next step (double-buffered
workspace); consecutive steps are chained by programmatic dependent launch.

Secondary workload (configs[4] shape, C5): a sweep of synthetic scenarios
replayed end to end per step (arrivals -> replay -> SLO -> features +
3 predictors), reported as scenario replays/s.

Multi-GPU (torchrun, one rank per GPU, NCCL): decisions and scenarios shard
across ranks with no data-path collective (weak scaling); per-rank times are
reduced with MAX.  `--impl reference` times the CPU oracle port on the host
cores instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEC = 32
CAP = 4
ALPHA = 0.5
C4_PASSES = 4  # replay + verify passes queued per long trace (3 needed at slow 2.0, min_len 96)
REPLAY_SCEN = 10000  # BASELINE configs[4]: a sweep of 10^4 synthetic scenarios (per GPU)
METRIC = "candidate co-location predictions/sec and scenario replays/sec at 1/2/4/8 B200"


def _env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(kernel: str):
    """ncu dram bytes (read + write) per launch of `kernel` from the committed
    `ncu --set full` summary (profiles/ncu_summary.json), if present."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    return None


def cpu_model() -> str:
    """Host CPU model and usable cores (every cpu_baseline carries it)."""
    name = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                name = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{name}, {len(os.sched_getaffinity(0))} cores available"


def one_thread_blas():
    """Context: numpy's BLAS/LAPACK pinned to one thread (the reference as shipped)."""
    from threadpoolctl import threadpool_limits

    return threadpool_limits(limits=1)


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def wait_first(self, timeout: float = 5.0):
        """Block until nvidia-smi has written its first sample."""
        t0 = time.time()
        while self.p is not None and time.time() - t0 < timeout:
            if os.path.getsize(self.f.name) > 0:
                return
            time.sleep(0.05)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[0]) for r in rows if len(r) >= 7 and r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 7 and r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 7 for i in range(4) if r[3 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------- workloads
def decision_coefs(n_dec: int) -> np.ndarray:
    """[n_dec][2][7]: coarse (static) / fine (EWMA 1/2) OLS refits on growing
    windows of the bundled trace's samples (`sweep.c2_decision_coefs`)."""
    from paper_2512_18725_b200.sweep import c2_decision_coefs

    return c2_decision_coefs(n_dec, ALPHA)


def cpu_candidate_rate(table, W, seconds: float, seed: int = 0):
    """Oracle port (`oracle.candidate_predictions`, restated from the
    reference's functions) on a sample of cap-4 candidates, one core."""
    import itertools

    import oracle as O

    rng = np.random.default_rng(seed)
    E = len(table.solo)
    sets = [()]
    for k in range(1, CAP):
        sets += list(itertools.combinations_with_replacement(range(E), k))
    n = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        for _ in range(200):
            o = int(rng.integers(E))
            pe = sets[int(rng.integers(len(sets)))]
            O.candidate_predictions(o, list(pe), table.solo, table.thr, W[0, 0], W[0, 1], ALPHA)
            n += 2
    dt = time.perf_counter() - t0
    return n / dt, n, dt


def cpu_replay_rate(table, seconds: float, start: int = 0):
    """The oracle's C restatement of `run_scenario` (`simcore.py:218-310`,
    literal heap engine) + its arrival generator + the numpy restatement of
    the coarse / fine / adaptive evaluation (`oracle.scenario_eval`) on one
    core, over C5 scenarios start, start+1, ... until `seconds` elapse:
    (replays/s, n, s)."""
    import oracle as O
    from paper_2512_18725_b200.sweep import c5_scenario

    ta = table.arrays()
    otab = O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr)
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        spec = c5_scenario(table, start + n)
        O.scenario_eval(O.run_scenario(spec, otab), spec, otab)  # replay + coarse / fine / adaptive evaluation
        n += 1
    dt = time.perf_counter() - t0
    return n / dt, n, dt


def _ref_replay_worker(args):
    seconds, start = args
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles

    return cpu_replay_rate(gen_synthetic_profiles(), seconds, start)[1]


def _ref_worker(args):
    seconds, seed = args
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles

    table = gen_synthetic_profiles().arrays()
    W = np.random.default_rng(7).normal(0, 0.3, size=(1, 2, 7))
    return cpu_candidate_rate(table, W, seconds, seed)[1]


REFIT_STREAMS = 10000
REFIT_LEN = 300
OLS_ROWS = 1 << 24
REFIT_WINDOW = 64


def refit_secondary(a, stream, barrier, max_over_ranks, rank) -> dict:
    """C3 shape: prequential RLS / SGD over 10^4 concurrent streams of 300
    samples (`predict.py:157-205`), and the OLS statistics reduction over
    2^24 samples (56 B each, HBM-read bound, `predict.py:53-66`)."""
    import ctypes

    import torch
    from paper_2512_18725_b200 import _abi

    L = _abi.load()
    rng = np.random.default_rng(100 + rank)
    n = REFIT_STREAMS * REFIT_LEN
    X = torch.tensor(rng.uniform(0.0, 1.0, size=(n, 6)), device="cuda")
    w_true = np.array([0.3, 0.5, 0.2, 0.8, 1.1, 0.4])
    y = torch.tensor(X.cpu().numpy() @ w_true + 1.0 + 0.02 * rng.standard_normal(n), device="cuda")
    off = torch.arange(0, n + 1, REFIT_LEN, dtype=torch.int64, device="cuda")
    params0 = torch.zeros(REFIT_STREAMS, 7, dtype=torch.float64, device="cuda")
    P0 = (100.0 * torch.eye(7, dtype=torch.float64, device="cuda")).repeat(REFIT_STREAMS, 1, 1).contiguous()
    lam = torch.full((REFIT_STREAMS,), 0.99, dtype=torch.float64, device="cuda")
    eta = torch.full((REFIT_STREAMS,), 0.01, dtype=torch.float64, device="cuda")
    pred = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.zeros(REFIT_STREAMS, dtype=torch.int32, device="cuda")
    s = stream.cuda_stream

    def run(kind):
        p = params0.clone()
        if kind == "rls":
            P = P0.clone()
            return lambda: _abi.check(L.intf_rls_streams(X.data_ptr(), y.data_ptr(), off.data_ptr(), REFIT_STREAMS,
                                                         lam.data_ptr(), p.data_ptr(), P.data_ptr(), pred.data_ptr(),
                                                         st.data_ptr(), s), "rls")
        return lambda: _abi.check(L.intf_sgd_streams(X.data_ptr(), y.data_ptr(), off.data_ptr(), REFIT_STREAMS,
                                                     eta.data_ptr(), p.data_ptr(), pred.data_ptr(), st.data_ptr(), s),
                                  "sgd")

    out = {}
    for kind in ("rls", "sgd"):
        f = run(kind)
        f()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f()
        e1.record(stream)
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1))
        out[kind] = {"updates_per_s": n / (ms / 1e3), "ms": ms}
    Xo = torch.rand(OLS_ROWS, 6, dtype=torch.float64, device="cuda")
    yo = torch.rand(OLS_ROWS, dtype=torch.float64, device="cuda")
    stats = torch.zeros(56, dtype=torch.float64, device="cuda")
    ws = torch.empty(_abi.OLS_WS_DOUBLES, dtype=torch.float64, device="cuda")
    for _ in range(3):
        _abi.check(L.intf_ols_stats(Xo.data_ptr(), yo.data_ptr(), OLS_ROWS, stats.data_ptr(), ws.data_ptr(), s), "ols")
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _abi.check(L.intf_ols_stats(Xo.data_ptr(), yo.data_ptr(), OLS_ROWS, stats.data_ptr(), ws.data_ptr(), s), "ols")
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    peak, _ = _peaks()
    gbs = 56.0 * OLS_ROWS / (ms / 1e3) / 1e9
    out["ols_stats"] = {"samples_per_s": OLS_ROWS / (ms / 1e3), "ms": ms, "achieved_gbs": gbs, "frac": gbs / peak,
                        "bytes_per_sample": 56}
    # refit each window (configs[2]): fit_ols_xy on every REFIT_WINDOW-sample window, one launch (k_ols_windows_tma)
    n_win = (OLS_ROWS + REFIT_WINDOW - 1) // REFIT_WINDOW
    wparams = torch.empty(n_win * 7, dtype=torch.float64, device="cuda")
    winfo = torch.empty(n_win * 3, dtype=torch.int32, device="cuda")

    def windows():
        _abi.check(L.intf_ols_windows(Xo.data_ptr(), yo.data_ptr(), OLS_ROWS, REFIT_WINDOW, None,
                                      wparams.data_ptr(), winfo.data_ptr(), s), "ols_windows")

    for _ in range(3):
        windows()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    windows()
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    gbs = 56.0 * OLS_ROWS / (ms / 1e3) / 1e9
    out["ols_windows"] = {"fits_per_s": n_win / (ms / 1e3), "samples_per_s": OLS_ROWS / (ms / 1e3), "ms": ms,
                          "window": REFIT_WINDOW, "fits": n_win, "achieved_gbs": gbs, "frac": gbs / peak,
                          "ridge_windows": int((winfo.view(-1, 3)[:, 0] != 0).sum().item())}
    out["workload"] = (f"{REFIT_STREAMS} concurrent prequential streams x {REFIT_LEN} samples (RLS lambda 0.99, "
                       f"SGD eta 0.01, fp64); OLS Z^T Z / Z^T y over {OLS_ROWS} samples; refit each window of "
                       f"{REFIT_WINDOW} samples over the same {OLS_ROWS} samples")
    return out


C4_REQUESTS = 1e6


def c4_secondary(a, stream, barrier, max_over_ranks, rank, world) -> dict:
    """C4 shape: one 10^6-request, 16-model (bs <= 64, cap 4) trace replayed
    with busy-period sharding (speculative idle boundaries planned, verified
    and merged on the device; C4_PASSES passes queued with device-side job
    counts, one host read per trace, inside the timed region).  N > 1: the
    SAME trace sharded across the ranks (c4_sharded).  Also at N = 1:
    back-to-back replays of the trace on four buffer sets and streams, two
    each (`pipelined`: repeated replays of one trace, each checked complete)."""
    import torch
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.sweep import c4_scenario, table16

    t16, arch = table16()
    spec = c4_scenario(t16, arch, n_requests=C4_REQUESTS, seed=1)  # ONE trace, the same on every rank
    ta = t16.arrays()
    if world > 1:
        return c4_sharded(a, spec, ta, stream, barrier, max_over_ranks, rank, world)
    n_c4_pipes = int(os.environ.get("INTF_BENCH_C4_PIPES", "4"))  # buffer sets / streams in flight (profiles/c4_pipes_r1m.txt)
    pipes = [engine.ReplayPipeline([spec], ta, scale=1.2) for _ in range(n_c4_pipes)]
    for p in pipes:  # warm-up (also sizes the job scratch); default slow 2.0, min_len 96
        engine.replay_segmented(p, passes=C4_PASSES)
    pipe = pipes[0]
    barrier()
    # one trace: C4_PASSES replay + verify passes queued with device-side job
    # counts, one host read at the end (more passes if ever needed)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    stats = engine.replay_segmented(pipe, passes=C4_PASSES)
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    n_req = int(pipe.t["n_req"][0].item())
    st = int(pipe.t["status"][0].item())
    # back-to-back traces on n_c4_pipes buffer sets and streams (each trace fully
    # stream-ordered: its low-parallelism phases overlap the other's work);
    # every trace's pending-job count is kept and checked after the timing
    K = 2 * n_c4_pipes
    rstreams = [torch.cuda.Stream() for _ in pipes]
    pending = torch.zeros(K, dtype=torch.int32, device="cuda")
    fins = []
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    p0.record(stream)
    for rs in rstreams:
        rs.wait_stream(stream)
    for k in range(K):
        q = k % n_c4_pipes
        with torch.cuda.stream(rstreams[q]):
            fins.append(engine.replay_segmented(pipes[q], passes=C4_PASSES, stats=False))
            pending[k:k + 1].copy_(pipes[q]._jobs.t["todo_count"][:1])
    for rs in rstreams:
        stream.wait_stream(rs)
    p1.record(stream)
    barrier()
    pms = max_over_ranks(p0.elapsed_time(p1)) / K
    complete = int(pending.sum().item()) == 0 and all(int(p.t["status"][0].item()) == 0 for p in pipes)
    for f in fins[-n_c4_pipes:]:
        f()
    stage = c4_stages(pipe)
    peak, _ = _peaks()
    fs_ms = stage["formation+noise"] + stage["slo"]
    stage_roofline = {"stages": "formation (+ noise table) + SLO report", "algorithmic_bytes_per_request": 23,
                      "achieved_gbs": 23.0 * n_req / (fs_ms / 1e3) / 1e9, "peak": peak,
                      "frac": 23.0 * n_req / (fs_ms / 1e3) / 1e9 / peak}
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        # the oracle's C heap-engine replay of the same trace (+ its arrivals), one core, once
        import oracle as O

        t0 = time.perf_counter()
        ref = O.run_scenario(spec, O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr))
        dt = time.perf_counter() - t0
        cpu = {"value": len(ref["arr_t"]) / dt, "unit": "requests/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
               "sample": f"the whole {len(ref['arr_t'])}-request trace (oracle C replay: heap engine + arrivals) "
                         f"in {dt:.2f} s"}
    return {"metric": "requests replayed/sec (single long trace)", "value": world * n_req / (ms / 1e3),
            "unit": "requests/s", "ms_per_trace": ms, "requests": n_req, "status": st, **stats,
            "pipelined": {"value": world * n_req / (pms / 1e3), "unit": "requests/s", "ms_per_trace": pms,
                          "traces": K, "streams": n_c4_pipes, "complete": complete},
            "cpu_baseline": cpu, "stage_ms": stage, "stage_roofline": stage_roofline,
            "workload": "C4: 16 models (6 default + 10 rng(123) archetypes), bs 1-64, cap 4, window U(10,20) ms, "
                        "sigma 0.05, total rho 0.5 at bs 64; one trace per GPU; arrivals + formation + noise + "
                        "busy-period-sharded replay + SLO + features"}


def c4_stages(pipe) -> dict:
    """One extra (untimed) pass of the long-trace path with events between its
    launches: per-stage device time in ms (`tools/c4_breakdown.py`)."""
    import ctypes

    import torch
    from paper_2512_18725_b200 import _abi

    L, st = pipe.lib, torch.cuda.current_stream().cuda_stream
    bt, B = ctypes.byref(pipe.batch), ctypes.byref(pipe.B)
    J, tab = ctypes.byref(pipe._jobs.J), ctypes.byref(pipe.dtable.struct)
    marks = []

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((name, e))

    mark("start")
    _abi.check(L.intf_generate_arrivals(bt, B, st), "arrivals")
    mark("arrivals")
    _abi.check(L.intf_form_batches(bt, B, st), "formation")
    mark("formation+noise")
    _abi.check(L.intf_jobs_plan(bt, tab, B, J, st), "plan")
    mark("plan")
    total = int(pipe._jobs.J.total_slots)
    for _ in range(C4_PASSES):
        _abi.check(L.intf_jobs_replay(bt, tab, B, J, -total, st), "jobs replay")
        _abi.check(L.intf_jobs_verify(bt, B, J, st), "jobs verify")
    mark("replay+verify passes")
    pipe.run_slo_features(slo=True, features=False)
    mark("slo")
    pipe.run_slo_features(slo=False, features=True)
    mark("features")
    torch.cuda.synchronize()
    return {b: ea.elapsed_time(eb) for (_, ea), (b, eb) in zip(marks, marks[1:])}


def c4_sharded(a, spec, ta, stream, barrier, max_over_ranks, rank, world) -> dict:
    """C4 at N > 1: the one 10^6-request trace sharded across the ranks
    (distributed.replay_trace_sharded: replicated arrivals / formation / job
    plan, each rank replays the jobs starting in its batch range, job results
    MAX-all_reduced before every verification pass, the owned per-batch
    outputs SUM-all_reduced at the end, SLO report on every rank).  Strong
    scaling: the same trace for every N; time = max over ranks."""
    import torch
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.distributed import replay_trace_sharded

    pipe = engine.ReplayPipeline([spec], ta, scale=1.2)
    for _ in range(2):
        replay_trace_sharded(pipe, passes=C4_PASSES, backend=a.backend)
    barrier()
    reps = 4
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        stats = replay_trace_sharded(pipe, passes=C4_PASSES, backend=a.backend)
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / reps
    n_req = int(pipe.t["n_req"][0].item())
    return {"metric": "requests replayed/sec (single long trace)", "value": n_req / (ms / 1e3), "unit": "requests/s",
            "ms_per_trace": ms, "requests": n_req, "status": int(pipe.t["status"][0].item()), "scaling": "strong",
            **stats, "cpu_baseline": None,
            "workload": "C4: ONE trace (16 models, bs 1-64, cap 4, seed 1) sharded over the ranks: replicated "
                        "arrivals + formation + job plan, jobs replayed by the rank owning their first batch, "
                        "MAX all_reduce of job results per verify pass, SUM all_reduce of the owned per-batch "
                        "outputs, SLO report on every rank"}


def prep_kernel_ms(scorer, stream) -> float:
    """k_cand_prep alone on the current stream (context for step_kernels)."""
    import torch

    for _ in range(3):
        scorer.prepare()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        scorer.prepare()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10


def replay_stage_times(pipe, stream) -> dict:
    """One extra (untimed) pass of the replay pipeline with events between
    its launches: per-stage device time in ms."""
    import ctypes

    import torch
    from paper_2512_18725_b200 import _abi

    L, s = _abi.load(), stream.cuda_stream
    bt, B = ctypes.byref(pipe.batch), ctypes.byref(pipe.B)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    ev[0].record(stream)
    _abi.check(L.intf_generate_arrivals(bt, B, s), "arrivals")
    ev[1].record(stream)
    _abi.check(L.intf_form_batches(bt, B, s), "formation")  # timed on its own (intf_replay forms again)
    ev[2].record(stream)
    _abi.check(L.intf_replay(bt, ctypes.byref(pipe.dtable.struct), B, s), "replay")
    ev[3].record(stream)
    pipe.run_slo_features(slo=True, features=False, evaluate=False)
    ev[4].record(stream)
    pipe.run_slo_features(slo=False, features=True, evaluate=False)
    ev[5].record(stream)
    if pipe.evaluate is not None:
        pipe.run_evaluation()
    ev[6].record(stream)
    torch.cuda.synchronize()
    names = ["arrivals", "formation+noise", "replay", "slo", "features", "evaluation"]
    return {n: ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(names)}


def c5_sweep(a, stream, barrier, max_over_ranks, rank, world, dist, table, W, scorer=None) -> dict:
    """C5 (BASELINE configs[4]): a FIXED sweep of 10^4 synthetic scenarios
    (default_rng([2512, i])) split over the ranks by expected requests
    (lambda*T, longest-processing-time first; strong scaling).  One step = the
    whole sweep: arrivals -> formation -> noise -> replay (warp per scenario)
    -> SLO -> features (static + EWMA(1/2)) -> per scenario the coarse / fine
    / adaptive evaluation (75/25 chronological split, OLS fits, RLS
    prequential tail, 3 EvalReports) -> the per-scenario rows gathered
    (NCCL all_gather, N > 1).  Consecutive sweeps run on several pipelines
    (buffer sets on their own streams), so one sweep's short stages overlap
    the longest scenarios' replay chains of the previous ones."""
    import torch
    from paper_2512_18725_b200 import _abi, engine
    from paper_2512_18725_b200.distributed import SweepRows, gather_sweep_rows, lpt_shards
    from paper_2512_18725_b200.sweep import c5_scenarios, expected_requests

    ta = table.arrays()
    specs_all = c5_scenarios(table, REPLAY_SCEN)
    shards = lpt_shards([expected_requests(sp) for sp in specs_all], world)
    mine = shards[rank]
    specs = [specs_all[i] for i in mine]
    counts = [len(sh) for sh in shards]
    preds = [_abi.Predictor(ewma=0, alpha=1.0, w=tuple(W[-1, 0])), _abi.Predictor(ewma=1, alpha=ALPHA, w=tuple(W[-1, 1]))]
    noise_k = int(os.environ.get("INTF_NOISE_K", engine.NOISE_K))  # tools/noise_k.sh sweeps it
    # in-flight sweeps: the step is bounded by its longest scenario's chain
    # (one warp), so fewer scenarios per GPU need more sweeps in flight
    n_pipes = int(os.environ.get("INTF_BENCH_PIPES", str(3 * world)))
    pipes = [engine.ReplayPipeline(specs, ta, preds=preds, scale=1.5, noise_k=noise_k, evaluate=(0, 1, 0.99))
             for _ in range(n_pipes)]
    rows = [SweepRows(p) for p in pipes]
    backend = a.backend
    for _ in range(max(1, a.warmup)):
        for p in pipes:
            p.run()
    barrier()
    st = pipes[0].status()
    gathered = [None] * n_pipes

    def step(k):
        q = k % n_pipes
        pipes[q].run()
        loc = rows[q].build()
        gathered[q] = gather_sweep_rows(loc, counts, backend) if dist is not None else [loc]

    rstreams = [torch.cuda.Stream() for _ in pipes]
    for k in range(n_pipes):  # warm every pipeline's full step on its own stream (row build + gather allocations)
        with torch.cuda.stream(rstreams[k]):
            step(k)
    barrier()
    r_steps = max(n_pipes, a.steps)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    for rs in rstreams:
        rs.wait_stream(stream)
    for k in range(r_steps):
        with torch.cuda.stream(rstreams[k % n_pipes]):
            step(k)
    for rs in rstreams:
        stream.wait_stream(rs)
    r1.record(stream)
    barrier()
    rep_ms = max_over_ranks(r0.elapsed_time(r1)) / r_steps
    pipe = pipes[0]
    stage_ms = replay_stage_times(pipe, stream)
    n_batches = int(pipe.t["n_batches"][: pipe.pb.n_scen].sum().item())
    n_req = int(pipe.t["n_req"][: pipe.pb.n_scen].sum().item())
    est = pipe.eval_status.cpu().numpy()
    # the longest scenario replayed alone: the floor of a sweep's time on one GPU
    heavy = engine.ReplayPipeline(specs[:1], ta, preds=preds, scale=1.5, noise_k=noise_k, evaluate=(0, 1, 0.99))
    for _ in range(2):
        heavy.run()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    heavy.run()
    t1.record(stream)
    torch.cuda.synchronize()
    tail_ms = t0.elapsed_time(t1)
    decisions = real_decisions(stream, barrier, max_over_ranks, scorer, pipe, W) if scorer is not None else None
    summary = None
    if rank == 0:  # untimed: the sweep's result, every scenario in index order
        allrows = np.full((REPLAY_SCEN, gathered[0][0].shape[1]), np.nan)
        for r, blk in enumerate(gathered[(r_steps - 1) % n_pipes]):
            allrows[np.asarray(shards[r])] = blk.cpu().numpy()
        summary = sweep_summary(allrows)
    return {"metric": "scenario replays/sec (incl. coarse / fine / adaptive evaluation)",
            "value": REPLAY_SCEN / (rep_ms / 1e3), "unit": "replays/s", "ms_per_step": rep_ms, "scaling": "strong",
            "scenarios_total": REPLAY_SCEN, "scenarios_this_gpu": len(specs), "pipelines": n_pipes,
            "requests": n_req, "batches": n_batches, "status_nonzero": int(np.count_nonzero(st)),
            "eval_invalid": int(np.count_nonzero(est[: len(specs)] & 1)),
            "tail_ms": tail_ms, "tail_scenario_batches": int(heavy.t["n_batches"][0].item()),
            "workload": "C5: 10^4 synthetic scenarios (default_rng([2512,i]), 2-4 models, 1 s, cap 1-3) split over "
                        "the GPUs by lambda*T (LPT); per step: arrivals + formation + noise + replay (warp per "
                        "scenario) + SLO + features + per-scenario coarse/fine/adaptive evaluation (75/25 split, "
                        "OLS x2, RLS prequential tail, 3 EvalReports) + per-scenario rows gathered to every rank "
                        f"(N > 1: NCCL all_gather); consecutive sweeps on {n_pipes} pipelines / streams",
            "steps_timed": r_steps, "stage_ms": stage_ms, "stage_roofline": c5_stage_roofline(stage_ms, n_req),
            "summary": summary, "decisions": decisions}


def c5_stage_roofline(stage_ms: dict, n_req: int) -> dict:
    """SURVEY §8d's HBM figure for formation + SLO (~23 B per request) against
    the stages' isolated device time (the noise table, RNG compute, is inside
    intf_form_batches and counted as formation time)."""
    peak, _ = _peaks()
    ms = stage_ms["formation+noise"] + stage_ms["slo"]
    gbs = 23.0 * n_req / (ms / 1e3) / 1e9
    return {"stages": "formation (+ noise table) + SLO report", "algorithmic_bytes_per_request": 23,
            "ms": ms, "achieved_gbs": gbs, "peak": peak, "frac": gbs / peak,
            "note": "per-scenario work of ~800 requests in ~300 batches: latency / issue bound, not HBM bound"}


def real_decisions(stream, barrier, max_over_ranks, scorer, pipe, W) -> dict:
    """C2 on REAL scheduling decisions ("the per-decision candidate
    set from C5 replays"): every dispatch of this rank's share of the sweep is
    a decision whose running set is a column of the cap-4 enumeration; every
    own row (48) is scored against it by both predictors and reduced to the
    best own row, plus the FIFO batch's prediction (intf_dispatch_sets +
    intf_score_decisions, features prepared once)."""
    import torch

    coefs = torch.tensor(W[-1], dtype=torch.float64, device="cuda").contiguous()
    scorer.prepare_decisions()
    rank_t, own_t = scorer.dispatch_decisions(pipe)
    best, chosen = scorer.score_decisions(coefs, rank_t, own_t)
    torch.cuda.synchronize()
    n_dec = int((rank_t >= 0).sum().item())
    reps = 10
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        rank_t, own_t = scorer.dispatch_decisions(pipe)
        scorer.score_decisions(coefs, rank_t, own_t, best, chosen)
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / reps
    bk = best.cpu().numpy().view(np.uint64).reshape(-1, 2)
    valid = rank_t.cpu().numpy() >= 0
    hi = (bk[valid, 1] >> np.uint64(32)).astype(np.uint32)
    best_fine = np.where(hi >> np.uint32(31), hi & np.uint32(0x7FFFFFFF), ~hi).astype(np.uint32).view(np.float32)
    fifo_fine = chosen.cpu().numpy().reshape(-1, 2)[valid, 1]
    return {"metric": "real scheduling decisions scored/sec", "decisions": n_dec, "value": n_dec / (ms / 1e3),
            "unit": "decisions/s", "predictions_per_s": n_dec * 2 * scorer.E / (ms / 1e3), "ms": ms,
            "mean_fine_prediction": {"fifo_batch": float(fifo_fine.mean()), "best_own_row": float(best_fine.mean())},
            "workload": "every dispatch of the replayed C5 sweep (this GPU's share): running set -> column of the "
                        "cap-4 enumeration; 48 own rows x {coarse, fine} scored, best own row + the FIFO batch's "
                        "prediction per decision (intf_dispatch_sets + intf_score_decisions)"}


def sweep_summary(rows: np.ndarray) -> dict:
    """SURVEY §8d C5 report: SLO satisfaction over scenarios (mean / median of
    the per-scenario request-weighted satisfaction) and, per predictor, the
    distribution of the per-scenario median relative error and MSE."""
    from paper_2512_18725_b200.distributed import REPORT_MODELS

    slo = rows[:, 18:].reshape(len(rows), REPORT_MODELS, 5)
    n, met = np.nansum(slo[..., 0], axis=1), np.nansum(slo[..., 1], axis=1)
    sat = met / np.where(n > 0, n, np.nan)
    out = {"scenarios": int(len(rows)), "slo_satisfaction_mean": float(np.nanmean(sat)),
           "slo_satisfaction_median": float(np.nanmedian(sat))}
    for k, name in enumerate(("coarse", "fine", "adaptive")):
        rep = rows[:, 6 * k: 6 * k + 6]
        ok = rep[:, 5] > 0
        out[name] = {"scenarios": int(ok.sum()), "median_rel_p50": float(np.median(rep[ok, 2])),
                     "mean_rel_p50": float(np.mean(rep[ok, 2])), "median_rel_p95": float(np.median(rep[ok, 4])),
                     "median_mse": float(np.median(rep[ok, 0]))}
    return out


def c1_leg(a, stream, barrier, max_over_ranks, rank, world, W) -> dict:
    """C1 (BASELINE configs[0]): the reference's bundled trace
    `mixed_three_model.json` at seed 7 (3 models, cap 2; 3,789 requests, 1,528
    batches), static features, the coarse predictor.  Device: one replay
    pipeline pass (arrivals -> formation -> noise -> replay -> SLO ->
    features -> forward), CUDA events, >= 20 repetitions.  e2e: the public
    API call a user makes -- `run_scenario(spec, table)` (H2D of the scenario,
    every result materialised as the reference's objects) + `predict_many` of
    its samples.  CPU: the oracle's C heap-engine replay + numpy features and
    forward of the same trace on one core.  Replicas only across GPUs (one
    trace does not shard)."""
    import torch
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import _abi, engine
    from paper_2512_18725_b200.predict import LinearModel, predict_many
    from paper_2512_18725_b200.sweep import BUNDLED_SEED7
    from paper_2512_18725_b200.workload import scenario_from_dict

    table = p.gen_synthetic_profiles()
    ta = table.arrays()
    coarse = _abi.Predictor(ewma=0, alpha=1.0, w=tuple(W[-1, 0]))
    pipe = engine.ReplayPipeline([BUNDLED_SEED7], ta, preds=[coarse])
    reps = max(20, a.steps)

    def timed(f):
        for _ in range(5):
            f()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            f()
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1)) / reps

    warp_ms = timed(pipe.run)  # one warp replays the whole trace
    jpipe = engine.ReplayPipeline([BUNDLED_SEED7], ta, preds=[coarse])

    def jobs():  # the trace as speculative busy-period jobs, 3 device-queued passes, one host check
        engine.replay_segmented(jpipe, min_len=16, passes=3, stats=False)()

    ms = timed(jobs)
    nb = int(pipe.t["n_batches"][0].item())
    jv, wv = jpipe.scenario(jpipe.fetch(), 0), pipe.scenario(pipe.fetch(), 0)
    same = all(np.array_equal(jv[k], wv[k]) for k in ("order", "b_completion", "r_slo_met", "Yhat"))
    spec = scenario_from_dict(BUNDLED_SEED7)
    model = LinearModel(w=np.array(W[-1, 0, :6]), b=float(W[-1, 0, 6]))

    def api_call():
        res = p.run_scenario(spec, table)
        return res, predict_many(model, np.array([smp.x for smp in res.samples]))

    for _ in range(2):
        api_call()
    barrier()
    t0 = time.perf_counter()
    n_e2e = 10
    for _ in range(n_e2e):
        res, yhat = api_call()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / n_e2e)
    ok = len(res.outcomes) == nb == 1528 and len(res.records) == 3789 and bool(np.isfinite(yhat).all())
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        import oracle as O

        otab = O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr)
        with one_thread_blas():
            t0 = time.perf_counter()
            k = 0
            while time.perf_counter() - t0 < min(5.0, a.cpu_seconds) or k < 3:
                rep = O.run_scenario(BUNDLED_SEED7, otab)
                X, y, _ = O.samples_from_replay(rep, BUNDLED_SEED7, otab, False, 1.0)
                _ = X @ W[-1, 0, :6] + W[-1, 0, 6]
                k += 1
            dt = time.perf_counter() - t0
        cpu = {"value": k / dt, "unit": "replays/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
               "sample": f"{k} replays of the bundled trace (oracle C heap engine + arrivals, numpy static "
                         f"features + forward) in {dt:.2f} s; the reference's own Python run_scenario: "
                         f"270.5 ms/replay on one core of the build container (SURVEY §6)"}
    return {"metric": "bundled-trace replays/sec (C1)", "value": world * 1e3 / ms, "unit": "replays/s",
            "us_per_replay": 1e3 * ms, "us_per_replay_one_warp": 1e3 * warp_ms, "jobs_equal_one_warp": same,
            "scaling": "weak (replicas only: one trace does not shard)",
            "batches": nb, "consistent": ok,
            "e2e": {"value": world * 1e3 / e2e_ms, "unit": "replays/s", "ms_per_call": e2e_ms,
                    "call": "run_scenario(spec, table) + predict_many (objects materialised on the host)",
                    "h2d_bytes_per_step": int(pipe.d_scen.numel() + pipe.d_models.numel()),
                    "d2h_bytes_per_step": int(sum(v.numel() * v.element_size() for v in pipe.t.values()))},
            "cpu_baseline": cpu,
            "workload": "C1: pkg/scenarios/mixed_three_model.json, seed 7, static mode, coarse predictor "
                        "(bench C2 decision 31's refit); device pass = arrivals + formation + noise + replay as "
                        "busy-period jobs (min_len 16, 3 queued passes + one host check) + SLO + features + "
                        "forward; us_per_replay_one_warp = the same with one warp replaying the whole trace"}


def c3_leg(a, stream, barrier, max_over_ranks, rank, world) -> dict:
    """C3 (BASELINE configs[2]): the reference's drift experiment
    (`experiments.py:153-205`: 4 datasets, EWMA(1/2) features, OLS warm
    start, offline / SGD (eta 0.01) / RLS (lambda 0.99) prequential on 300
    test samples) for seeds 0..19, end to end through the package
    (`experiments.drift_experiments`: all seeds' 80 scenarios in one batched
    replay, fits / streams / reports as batched device launches).  CPU: the
    oracle's composition of the same functions (C replay + numpy) on one core.
    Seeds shard across ranks (no collective)."""
    import torch
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import experiments as ex

    table = p.gen_synthetic_profiles()
    seeds = list(range(20))[rank::world]
    bases = [ex.default_drift_base(table, s) for s in seeds]
    ex.drift_experiments(bases[:2], table)  # warm-up
    barrier()
    t0 = time.perf_counter()
    cells = ex.drift_experiments(bases, table)
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0)
    mean = ex.mean_drift_table(cells)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        import oracle as O

        ta = table.arrays()
        otab = O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr)
        with one_thread_blas():
            t1 = time.perf_counter()
            n_cpu = 0
            while n_cpu < 2:
                O.drift_experiment(ex.drift_specs(bases[n_cpu]), otab)
                n_cpu += 1
            cdt = time.perf_counter() - t1
        cpu = {"value": n_cpu / cdt, "unit": "seeds/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
               "sample": f"drift_experiment seeds 0..{n_cpu - 1} (oracle C replay + numpy OLS / SGD / RLS / "
                         f"EvalReports) in {cdt:.2f} s; the reference: 2.20 s per seed (SURVEY §6)",
               "updates": cpu_update_rates(min(2.0, a.cpu_seconds / 5))}
    return {"metric": "drift experiments/sec (C3, seeds 0..19)", "value": len(bases) * world / dt,
            "unit": "seeds/s", "s_per_seed": dt / len(bases), "seeds": 20, "scaling": "strong (seeds shard)",
            "mean_mse": {f"{k[0]}/{k[1]}": v for k, v in sorted(mean.items())},
            "e2e": {"value": len(bases) * world / dt, "unit": "seeds/s",
                    "call": "experiments.drift_experiments(bases, table) (public API, host objects out)"},
            "cpu_baseline": cpu,
            "workload": "C3: drift_experiment(default_drift_base(table, s)) for s = 0..19: per seed 4 replays "
                        "(training + 3 shifted test sets), EWMA(1/2) features, OLS warm start, offline / SGD / "
                        "RLS prequential on <= 300 test samples, MSE per (dataset, method)"}


def cpu_update_rates(seconds: float) -> dict:
    """1-core numpy rates of the reference's learners (`predict.py:75-154`):
    RLS / SGD updates/s (one prequential stream) and OLS samples/s (fit_ols_xy
    on 10^5 rows), as the oracle restates them."""
    import oracle as O

    rng = np.random.default_rng(0)
    X = rng.uniform(0, 1, size=(100000, 6))
    y = X @ np.array([0.3, 0.5, 0.2, 0.8, 1.1, 0.4]) + 1.0
    out = {}
    with one_thread_blas():
        for method in ("rls", "sgd"):
            n, t0 = 0, time.perf_counter()
            while time.perf_counter() - t0 < seconds:
                O.prequential(np.zeros(6), 0.0, X[:500], y[:500], method, P=100.0 * np.eye(7))
                n += 500
            out[f"{method}_updates_per_s"] = n / (time.perf_counter() - t0)
        t0 = time.perf_counter()
        O.fit_ols_xy(X, y)
        out["ols_samples_per_s"] = len(y) / (time.perf_counter() - t0)
    out["cpu"] = cpu_model()
    out["cores"] = 1
    return out


# -------------------------------------------------------------- reference
def reference_arm(a):
    rank, world, _ = _env()
    if rank != 0:
        return 0
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    per_step = 1.0
    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(a.warmup):
            pool.map(_ref_worker, [(0.2, s) for s in range(cores)])
        times, preds = [], 0
        for k in range(a.steps):
            t0 = time.perf_counter()
            n = sum(pool.map(_ref_worker, [(per_step, 1000 * k + s) for s in range(cores)]))
            times.append(time.perf_counter() - t0)
            preds += n
        # scenario replays on every core (context; the driver's ratio uses `value`)
        t0 = time.perf_counter()
        n_rep = sum(pool.map(_ref_replay_worker, [(per_step, 100000 * (s + 1)) for s in range(cores)]))
        rep_rate = n_rep / (time.perf_counter() - t0)
    tot = sum(times)
    v = preds / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "predictions/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 candidate sets, cap 4 over the 48 bundled profile entries, coarse+fine "
                               "predictors (bounded random sample of candidates per step)", "cap": CAP},
        "cpu_baseline": {"value": v, "unit": "predictions/s", "cores": cores, "kind": "port", "cpu": cpu_model(),
                         "sample": f"{per_step:.1f} s of random cap-4 candidates per core per step "
                                   f"(oracle.candidate_predictions, reference functions restated)"},
        "e2e": {"value": v, "unit": "predictions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "replay": {"metric": "scenario replays/sec", "value": rep_rate, "unit": "replays/s", "cores": cores,
                   "sample": f"{n_rep} C5 scenarios (oracle C replay: heap engine + arrivals; numpy coarse/fine/"
                             f"adaptive evaluation), {per_step:.1f} s per core"},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------- product
def product_arm(a):
    import torch

    rank, world, local = _env()
    if a.backend == "gloo":  # plumbing test on a box with fewer GPUs than ranks (not a measurement)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if a.backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2512_18725_b200 import _abi, engine
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles
    from paper_2512_18725_b200.sweep import c5_scenarios, lpt_order

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if a.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    table = gen_synthetic_profiles()
    ta = table.arrays()
    W = decision_coefs(N_DEC)
    W = W * (1.0 + 1e-3 * rank)  # each rank scores its own decisions (weak scaling)
    scorer = engine.CandidateScorer(ta, cap=CAP, alpha=ALPHA)
    coefs = torch.tensor(W, dtype=torch.float64, device="cuda").contiguous()
    # two output buffers, alternated per step: each step's 256 MB must really
    # reach HBM (rewriting one buffer lets L2 absorb part of the next step)
    outs = [scorer.alloc(N_DEC), scorer.alloc(N_DEC)]
    out = outs[0]
    n_pred = N_DEC * 2 * scorer.n_cand  # useful predictions per step (row padding excluded)
    n_elems = scorer.out_elems(N_DEC)
    stream = torch.cuda.current_stream()

    # ---- device-resident timed region (clocks sampled across every timed region)
    clocks = Clocks(local)
    clocks.wait_first()
    # one step = forward of every candidate for this step's decisions + the
    # candidate-feature build for the next step (double-buffered workspace),
    # both in ONE k_cand_step launch (--side-stream: k_cand_stream + k_cand_prep
    # on a side stream).  The first step's features are built in warm-up and
    # the last timed step's feature build is joined before t_end, so the timed
    # region holds exactly K forward passes and K feature builds.
    scorer.pipeline_start(fused=not a.side_stream)
    for k in range(a.warmup):
        scorer.pipeline_step(coefs, outs[k & 1])
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(a.steps):
        scorer.pipeline_step(coefs, outs[k & 1])
    scorer.pipeline_join()
    t_end.record(stream)
    barrier()
    ms_total = max_over_ranks(t_start.elapsed_time(t_end))
    # per-launch duration of the step kernel with events around every launch
    # (a separate pass: events between launches would serialise the
    # programmatic dependent launches of the timed loop)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    for k in range(a.steps):
        scorer.pipeline_step(coefs, outs[k & 1], kernel_events=ev[k])
    scorer.pipeline_join()
    torch.cuda.synchronize()
    kern_ms = float(np.mean([s.elapsed_time(e) for s, e in ev]))
    prep_ms = prep_kernel_ms(scorer, stream)  # k_cand_prep alone (untimed pass)
    ms_step = ms_total / a.steps
    value = world * n_pred / (ms_step / 1e3)

    # ---- end to end through the host-buffer C-ABI calls: (1) the best
    # candidate per (decision, kind, own) -- what a scheduling decision
    # consumes: every candidate is scored, 24 KB of keys come back
    # (intf_best_candidates_host); (2) every prediction materialised on the
    # host (intf_predict_candidates_host, PCIe-bound: 256 MB per step)
    h_coefs = torch.tensor(W, dtype=torch.float64).pin_memory()
    hc = h_coefs.numpy()
    h_best = torch.empty(2 * N_DEC * scorer.E, dtype=torch.int64).pin_memory()
    hb = h_best.numpy().view(np.uint64)
    bscratch = torch.empty(scorer.best_scratch_elems(N_DEC) + scorer.ws_elems, dtype=torch.float32, device="cuda")

    def best_call():  # decision after decision: each call builds the next call's features in its launch
        scorer.best_host_pipelined(hc, hb, bscratch, sync=True)  # returns with the keys on the host

    def best_call_async():  # the asynchronous form + a stream synchronisation by the caller
        scorer.best_host_pipelined(hc, hb, bscratch)
        stream.synchronize()

    e2e_steps = max(10, a.steps)
    e2e_times = {}
    for name, fn in (("async", best_call_async), ("sync", best_call)):
        for _ in range(max(3, a.warmup)):
            fn()
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            fn()
        e2e_times[name] = max_over_ranks((time.perf_counter() - t0) * 1e3 / e2e_steps)
    e2e_ms = e2e_times["sync"]
    bval, brank = scorer.decode_best(hb, N_DEC)
    ok_best = bool(np.isfinite(bval).all() and (brank < scorer.n_sets).all())
    h_out = torch.empty(n_elems, dtype=torch.float32).pin_memory()
    scratch = torch.empty(scorer.scratch_elems(N_DEC), dtype=torch.float32, device="cuda")
    ho = h_out.numpy()
    for _ in range(max(1, a.warmup)):
        scorer.score_host(hc, ho, scratch)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mat_steps = max(1, min(a.steps, 10))
    e0.record(stream)
    for _ in range(mat_steps):
        scorer.score_host(hc, ho, scratch)
    e1.record(stream)
    barrier()
    mat_ms = max_over_ranks(e0.elapsed_time(e1)) / mat_steps
    ok = bool(np.isfinite(ho[:1000]).all())
    del scratch, h_out
    # device-resident best steps (the reduction mode's own kernel time)
    bbufs = [scorer.alloc_best(N_DEC) for _ in range(2)]
    scorer.pipeline_start(fused=True)
    for k in range(a.warmup):
        scorer.best_step(coefs, bbufs[k & 1], bbufs[(k + 1) & 1])
    barrier()
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b0.record(stream)
    for k in range(a.steps):
        scorer.best_step(coefs, bbufs[k & 1], bbufs[(k + 1) & 1])
    b1.record(stream)
    barrier()
    best_ms = max_over_ranks(b0.elapsed_time(b1)) / a.steps

    # ---- secondary: scenario replay sweep (C5: 10^4 scenarios, coarse / fine / adaptive)
    sweep = c5_sweep(a, stream, barrier, max_over_ranks, rank, world, dist, table, W, scorer)

    refit = refit_secondary(a, stream, barrier, max_over_ranks, rank)
    bundled = c1_leg(a, stream, barrier, max_over_ranks, rank, world, W)
    drift = c3_leg(a, stream, barrier, max_over_ranks, rank, world)
    longtrace = c4_secondary(a, stream, barrier, max_over_ranks, rank, world) if not a.no_c4 else None
    clk = clocks.stop()

    # ---- CPU baseline (rank 0, N=1 only): oracle port on a bounded sample
    cpu = replay_cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        rate, n, dt = cpu_candidate_rate(ta, W, a.cpu_seconds)
        cpu = {"value": rate, "unit": "predictions/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
               "sample": f"{n} predictions ({n // 2} random cap-4 candidates x coarse+fine, 1 decision) in {dt:.1f} s"}
        rrate, rn, rdt = cpu_replay_rate(table, min(5.0, a.cpu_seconds))
        replay_cpu = {"value": rrate, "unit": "replays/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
                      "sample": f"{rn} C5 scenarios (oracle C replay: heap engine + arrivals; numpy evaluation: "
                                f"split, 2 lstsq fits, RLS tail, 3 EvalReports) in {rdt:.1f} s"}

    # context: a pure device write (torch fill) of the same size, alternating
    # two buffers like the timed loop -- the write-only ceiling on this part
    for k in range(3):
        outs[k & 1].fill_(1.0)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for k in range(10):
        outs[k & 1].fill_(1.0)
    f1.record(stream)
    torch.cuda.synchronize()
    fill_gbs = 4.0 * n_elems * 10 / (f0.elapsed_time(f1) / 1e3) / 1e9

    peak, peak_src = _peaks()
    bytes_per_launch = 4.0 * n_pred  # implicit enumeration: fp32 output only
    fused = not a.side_stream
    kname = "k_cand_step" if fused else "k_cand_stream"
    # fused: every step is ONE k_cand_step launch, chained by programmatic
    # dependent launch, so the steady-state launch duration is this rank's
    # timed-region time / K; events around each launch (kern_ms) serialise
    # the chain and are reported as the isolated figure
    launch_ms = t_start.elapsed_time(t_end) / a.steps if fused else kern_ms
    achieved = bytes_per_launch / (launch_ms / 1e3) / 1e9
    traffic = _traffic(kname)
    line = {
        "metric": METRIC, "value": value, "unit": "predictions/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 forward (f64 features)", "data": "synthetic",
        "config": {"workload": "C2: all candidate co-location sets (cap 4, 48 bundled profile entries = 999,600 "
                               "candidates) x {coarse static, fine EWMA(1/2)} predictors x 32 refit decisions per "
                               "step per GPU; output fp32", "global_batch": n_pred * world,
                   "parallelism": f"dp{world} (decisions sharded, no collective)", "l2": "output 256 MB/step > L2; two output buffers alternated per step"},
        "e2e": {"value": world * n_pred / (e2e_ms / 1e3), "unit": "predictions/s", "ms_per_call": e2e_ms,
                "h2d_bytes_per_step": int(W.size * 8), "d2h_bytes_per_step": int(8 * 2 * N_DEC * scorer.E),
                "call": "intf_best_candidates_host_sync (pinned host buffers, host-timed, returns with the keys "
                        "in host memory): every candidate scored, the best per (decision, kind, own) returned; ONE "
                        "kernel launch per call -- the coefficients travel as a kernel parameter, the last block "
                        "writes the keys into the pinned buffer and a completion word the call spins on; each call "
                        "also builds the next call's candidate features (the fused step)", "valid": ok_best,
                "async_ms_per_call": e2e_times["async"],
                "materialized": {"value": world * n_pred / (mat_ms / 1e3), "unit": "predictions/s",
                                 "call": "intf_predict_candidates_host (every fp32 prediction to the host)",
                                 "d2h_bytes_per_step": int(4 * n_elems), "finite": ok,
                                 "pcie_gbs": (W.size * 8 + 4 * n_elems) / (mat_ms / 1e3) / 1e9}},
        "best_step": {"value": world * n_pred / (best_ms / 1e3), "unit": "predictions/s", "ms_per_step": best_ms,
                      "kernel": "k_cand_step<best> (device-resident, PDL-chained, 24 KB of keys per step)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                                            "from the committed ncu --set full capture "
                                                            "(profiles/ncu_summary.json), not this run",
                     "peak_source": peak_src, "kernel": kname,
                     "kernel_ms": launch_ms, "kernel_ms_isolated": kern_ms,
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "step": ("one k_cand_step launch per step: forward of every candidate (stream blocks) + feature "
                              "build for the next step (prep blocks), PDL-chained" if fused else
                              "k_cand_stream + k_cand_prep of the next step on a side stream"),
                     "k_cand_prep_ms_alone": prep_ms,
                     "write_only_reference_gbs": fill_gbs},
        "cpu_baseline": cpu,
        "clocks": clk,
        "gpu_launches": a.steps if fused else 2 * a.steps,
        "replay": {**sweep, "cpu_baseline": replay_cpu},
        "refit": refit,
        "bundled_trace": bundled,
        "drift": drift,
        "long_trace": longtrace,
    }
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=20)  # (the C2 step settles after ~20 launches: 0.964 -> 0.976 of HBM)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 long-trace secondary measurement")
    ap.add_argument("--side-stream", action="store_true",
                    help="C2 step as two launches (feature build on a side stream) instead of one fused launch")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the multi-rank plumbing with ranks sharing GPUs (numbers meaningless)")
    a = ap.parse_args()
    if a.warmup < 3:
        a.warmup = 3
    if a.impl == "reference":
        return reference_arm(a)
    return product_arm(a)


if __name__ == "__main__":
    sys.exit(main())
