"""Multi-GPU plumbing for the hot path: one process per GPU,
torch.distributed (NCCL on B200s, gloo in CPU tests).

Only two exchange steps exist on this path:
  * OLS refit over samples sharded across ranks: every rank reduces its
    shard to the 56 fp64 normal-equation statistics (intf_ols_stats); the
    ranks exchange them with one all_gather and sum IN RANK ORDER, so every
    rank solves the identical 7x7 system (deterministic, unlike a ring
    all_reduce whose summation order depends on the topology);
  * the scenario sweep: each rank replays a contiguous range of scenarios
    and the fixed-size per-scenario report rows are gathered to every rank.
Candidate scoring and the RLS/SGD streams shard with no collective
(independent decisions / streams).
"""
from __future__ import annotations

import numpy as np
import torch

REPORT_MODELS = 4
REPORT_WIDTH = 4 + 5 * REPORT_MODELS  # n_req, n_batches, n_segments, status, then per model (n, met, p50, p95, p99)


def shard_range(n: int, rank: int, world: int) -> tuple:
    """Contiguous balanced [lo, hi) of n units for this rank."""
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def weighted_shards(weights, world: int) -> list:
    """Contiguous shards balanced by weight (e.g. expected requests
    lambda*T per scenario): greedy cut at multiples of total/world."""
    w = np.asarray(weights, dtype=float)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for k in range(1, world):
        cuts.append(int(np.searchsorted(cum, cum[-1] * k / world)))
    cuts.append(len(w))
    cuts = np.maximum.accumulate(np.array(cuts))
    return [(int(cuts[k]), int(cuts[k + 1])) for k in range(world)]


def lpt_shards(weights, world: int) -> list:
    """Longest-processing-time-first assignment of units to ranks: units in
    descending weight (e.g. expected requests lambda*T of a scenario), each to
    the rank with the least assigned weight so far (ties: lowest rank).
    Returns one index list per rank, each in descending weight (the replay's
    own LPT order).  Deterministic, so every rank computes the same split."""
    w = np.asarray(weights, dtype=float)
    order = sorted(range(len(w)), key=lambda i: (-w[i], i))
    load = np.zeros(world)
    out = [[] for _ in range(world)]
    for i in order:
        r = int(np.argmin(load))
        out[r].append(i)
        load[r] += w[i]
    return out


SWEEP_ROW = 18 + 5 * REPORT_MODELS  # per scenario: 3 x EvalReport (mse, p25, p50, p75, p95, n) + per-model SLO


class SweepRows:
    """Per-scenario report rows of a ReplayPipeline built on the device
    (the fixed-size struct gathered to rank 0): the coarse / fine
    / adaptive EvalReports (intf_scenario_eval) and per deployed model (n,
    met, p50, p95, p99), padded to REPORT_MODELS models."""

    def __init__(self, pipe):
        S = pipe.pb.n_scen
        idx = np.full((S, REPORT_MODELS), -1, dtype=np.int64)
        for s in range(S):
            sc = pipe.pb.scen[s]
            for m in range(min(sc.n_models, REPORT_MODELS)):
                idx[s, m] = sc.model_off + m
        self.pipe = pipe
        self.valid = torch.as_tensor(idx >= 0, device=pipe.dev)
        self.idx = torch.as_tensor(np.maximum(idx, 0), device=pipe.dev)
        self.rows = torch.zeros(S, SWEEP_ROW, dtype=torch.float64, device=pipe.dev)

    def build(self) -> torch.Tensor:
        """Enqueue the row build on the current stream; returns rows [S, SWEEP_ROW]."""
        p, S = self.pipe, self.pipe.pb.n_scen
        self.rows[:, :18] = p.eval_report.view(-1, 18)[:S]
        per = torch.stack([p.slo_n[self.idx].double(), p.slo_met[self.idx].double(),
                           p.slo_p.view(-1, 3)[self.idx, 0], p.slo_p.view(-1, 3)[self.idx, 1],
                           p.slo_p.view(-1, 3)[self.idx, 2]], dim=-1)
        per = torch.where(self.valid[..., None], per, torch.full_like(per, float("nan")))
        self.rows[:, 18:] = per.reshape(S, -1)
        return self.rows


def gather_sweep_rows(local: torch.Tensor, counts: list, backend: str = "nccl"):
    """all_gather of per-rank [n_r, F] row blocks (n_r = counts[r]): returns the
    list of every rank's block (padded blocks trimmed), on every rank."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [local]
    maxn = max(counts)
    pad = torch.full((maxn, local.shape[1]), float("nan"), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    if backend != "nccl":
        pad = pad.cpu()
    parts = [torch.empty_like(pad) for _ in counts]
    dist.all_gather(parts, pad)
    return [p[:n] for p, n in zip(parts, counts)]


def allreduce_ols_stats(stats: torch.Tensor) -> torch.Tensor:
    """Sum the 56 OLS statistics over ranks in rank order (all_gather)."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return stats
    parts = [torch.empty_like(stats) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, stats.contiguous())
    out = parts[0].clone()
    for p in parts[1:]:
        out += p
    return out


def report_rows(pipe, h) -> np.ndarray:
    """Fixed-size per-scenario report rows from a fetched ReplayPipeline."""
    S = pipe.pb.n_scen
    rows = np.full((S, REPORT_WIDTH), np.nan)
    for s in range(S):
        sc = pipe.pb.scen[s]
        rows[s, 0] = h["n_req"][s]
        rows[s, 1] = h["n_batches"][s]
        rows[s, 2] = h["n_segments"][s]
        rows[s, 3] = h["status"][s]
        for m in range(min(sc.n_models, REPORT_MODELS)):
            g = sc.model_off + m
            rows[s, 4 + 5 * m: 9 + 5 * m] = (h["slo_n"][g], h["slo_met"][g], *h["slo_p"][g])
    return rows


def gather_rows(local: torch.Tensor, n_total: int) -> torch.Tensor:
    """all_gather of per-rank [n_local, F] row blocks laid out by
    shard_range; returns the full [n_total, F] table on every rank."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    width = local.shape[1]
    maxn = max(shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0] for r in range(world))
    pad = torch.full((maxn, width), float("nan"), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([parts[r][: shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0]]
                      for r in range(world)])


def sweep(specs_all: list, table, preds=(), device_rows: bool = True):
    """Replay this rank's shard of a scenario sweep on its GPU and gather the
    report rows of all scenarios (C5 across GPUs)."""
    import torch.distributed as dist

    from . import engine

    rank = dist.get_rank() if dist.is_initialized() else 0
    world = dist.get_world_size() if dist.is_initialized() else 1
    lo, hi = shard_range(len(specs_all), rank, world)
    pipe, h = engine.run_batch(specs_all[lo:hi], table, preds=preds)
    local = torch.as_tensor(report_rows(pipe, h))
    if device_rows:
        local = local.cuda()
    return gather_rows(local, len(specs_all)).cpu().numpy()


# per-batch outputs of the replay that the owner of a batch writes (b_* by
# batch slot, out_order by outcome position = the same job ranges)
TRACE_GATHER = ("b_start", "b_completion", "b_measured", "b_nseg", "b_seg_off", "b_running", "out_order")


def _all_reduce(t: torch.Tensor, op, backend: str) -> None:
    import torch.distributed as dist

    if backend == "nccl":
        dist.all_reduce(t, op=op)
    else:  # gloo: host copies (tests / plumbing runs)
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)


def replay_trace_sharded(pipe, slow: float = 2.0, min_len: int = 96, passes: int = 4, slo: bool = True,
                         backend: str = "nccl", max_iters: int = 1000) -> dict:
    """ONE long trace (a single-scenario ReplayPipeline) replayed across the
    ranks: arrivals, batch formation and the speculative
    busy-period job plan are computed on every rank (identical, deterministic);
    the trace's batches are split into contiguous ranges, one per rank, and
    each rank replays only the jobs that start in its range
    (intf_jobs.own_lo/own_hi).  After every replay pass the job results (last
    completion, status/segment/reseat counts) are combined with an
    element-wise MAX all_reduce (non-owners hold -inf / 0), so every rank runs
    the same boundary verification and merges failing boundaries the same way
    -- a merged job belongs to the rank owning its first batch.  At the end
    each rank zeroes the per-batch outputs outside the batches of its final
    jobs and a SUM all_reduce assembles the whole trace on every rank, where
    the SLO report runs.  Bit-identical to the one-GPU replay."""
    import ctypes

    import torch.distributed as dist

    from . import _abi, engine

    if pipe.pb.n_scen != 1:
        raise ValueError("replay_trace_sharded shards one trace (a single-scenario pipeline)")
    rank = dist.get_rank() if dist.is_initialized() else 0
    world = dist.get_world_size() if dist.is_initialized() else 1
    L, st = pipe.lib, engine.stream_ptr()
    bt, B = ctypes.byref(pipe.batch), ctypes.byref(pipe.B)
    tab = ctypes.byref(pipe.dtable.struct)
    jobs = getattr(pipe, "_jobs", None)
    if jobs is None or jobs.key != (float(slow), int(min_len)):
        jobs = engine._DeviceJobs(pipe, slow, min_len)
        pipe._jobs = jobs
    J = ctypes.byref(jobs.J)
    _abi.check(L.intf_generate_arrivals(bt, B, st), "intf_generate_arrivals")
    _abi.check(L.intf_form_batches(bt, B, st), "intf_form_batches")
    for f in TRACE_GATHER:  # entries this rank does not own must be zero for the final SUM
        pipe.t[f].zero_()
    _abi.check(L.intf_jobs_plan(bt, tab, B, J, st), "intf_jobs_plan")
    nb = int(pipe.t["n_batches"][0].item())
    lo, hi = shard_range(nb, rank, world)
    jobs.J.own_lo = 0 if rank == 0 else lo
    jobs.J.own_hi = 2 ** 31 - 1 if rank == world - 1 else hi
    total = int(jobs.J.total_slots)
    need = total * pipe.pb.cap_max * pipe.seg_stride * 5
    if pipe.t["slot_seg"].numel() < need:
        pipe.t["slot_seg"] = torch.zeros(need, dtype=torch.float64, device=pipe.dev)
        pipe.B.slot_seg = pipe.t["slot_seg"].data_ptr()

    def one_pass(n_todo: int) -> None:
        _abi.check(L.intf_jobs_replay(bt, tab, B, J, n_todo, st), "intf_jobs_replay")
        if world > 1:
            _all_reduce(jobs.t["last"], dist.ReduceOp.MAX, backend)
            _all_reduce(jobs.t["info"], dist.ReduceOp.MAX, backend)
        _abi.check(L.intf_jobs_verify(bt, B, J, st), "intf_jobs_verify")

    n0 = int(jobs.t["n_jobs"][0].item())
    for _ in range(passes):  # queued with device-side job counts
        one_pass(-total)
    iters = passes
    while iters < max_iters:
        n = int(jobs.t["todo_count"][0].item())
        if n == 0:
            break
        one_pass(n)
        iters += 1
    # batches of this rank's final jobs: a contiguous range [first, last)
    nj = int(jobs.t["n_jobs"][0].item())
    jlo = jobs.t["lo"][:nj].cpu().numpy()
    jhi = jobs.t["hi"][:nj].cpu().numpy()
    mine = (jlo >= jobs.J.own_lo) & (jlo < jobs.J.own_hi)
    first, last = (int(jlo[mine].min()), int(jhi[mine].max())) if mine.any() else (0, 0)
    if world > 1:
        ro = pipe.pb.scen[0].req_off
        for f in TRACE_GATHER:
            t = pipe.t[f]
            t[: ro + first].zero_()
            t[ro + last:].zero_()
            _all_reduce(t, dist.ReduceOp.SUM, backend)
    if slo:
        pipe.run_slo_features(slo=True, features=False)
    return {"jobs_initial": n0, "jobs_final": nj, "iterations": iters, "batches": nb,
            "rank_batches": [first, last], "world": world}
