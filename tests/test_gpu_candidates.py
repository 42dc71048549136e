"""GPU parity of the candidate-set predictor (C2) against predictions
composed from reference functions (tests/golden/candidates_golden.npz) and
the oracle; fp32 output, tolerance 1e-5 relative."""
import numpy as np
import pytest
import torch

import oracle as O
from tests import _golden

pytestmark = pytest.mark.gpu
RTOL = 1e-5


def _scorer(cap, two_phase=True):
    from paper_2512_18725_b200 import engine

    return engine.CandidateScorer(_golden.table("default"), cap=cap, alpha=0.5, two_phase=two_phase)


def test_candidate_counts():
    from paper_2512_18725_b200 import engine

    assert [engine.candidate_count(48, c) for c in (2, 3, 4)] == [2352, 58800, 999600]


@pytest.mark.parametrize("cap,two_phase", [(2, True), (3, True), (2, False), (3, False)])
def test_candidates_match_reference_composition(cap, two_phase):
    from paper_2512_18725_b200 import engine

    C = _golden.load("candidates_golden.npz")
    sc = _scorer(cap, two_phase)
    coefs = torch.tensor(C["w"], dtype=torch.float64, device="cuda").reshape(1, 2, 7).contiguous()
    out = sc.alloc(1)
    sc.score(coefs, out)
    y = sc.view(out.cpu().numpy(), 1)[0]
    own, peers = C[f"cap{cap}/own"], C[f"cap{cap}/peers"]
    idx = np.array([engine.multiset_rank([q for q in pe if q >= 0], sc.E, cap) for pe in peers])
    np.testing.assert_allclose(y[0, own, idx], C[f"cap{cap}/y_coarse"], rtol=RTOL)
    np.testing.assert_allclose(y[1, own, idx], C[f"cap{cap}/y_fine"], rtol=RTOL)


@pytest.mark.parametrize("two_phase", [True, False])
def test_cap4_full_enumeration_sampled_against_oracle(two_phase):
    from paper_2512_18725_b200 import engine

    tab = _golden.table("default")
    sc = _scorer(4, two_phase)
    rng = np.random.default_rng(1)
    W = rng.normal(0, 0.5, size=(3, 2, 7))
    coefs = torch.tensor(W, dtype=torch.float64, device="cuda").contiguous()
    out = sc.alloc(3)
    sc.score(coefs, out)
    full = sc.view_full(out.cpu().numpy(), 3)
    assert np.all(full[..., sc.n_sets:] == 0)  # pad entries
    y = sc.view(out.cpu().numpy(), 3)
    assert np.isfinite(y).all()
    import itertools

    sets = [()]
    for k in range(1, 4):
        sets += list(itertools.combinations_with_replacement(range(sc.E), k))
    for _ in range(300):
        d, o, si = rng.integers(3), rng.integers(sc.E), rng.integers(len(sets))
        pe = sets[si]
        r = engine.multiset_rank(pe, sc.E, 4)
        yc, yf = O.candidate_predictions(int(o), list(pe), tab.solo, tab.thr, W[d, 0], W[d, 1], 0.5)
        np.testing.assert_allclose([y[d, 0, o, r], y[d, 1, o, r]], [yc, yf], rtol=RTOL, atol=1e-6)


def test_tiled_layout_roundtrip():
    """view_full inverts the tiled HBM layout: element (dec, kind, own, r) of the
    logical array is buffer[tile_off(dec, kind, own, r)] (csrc/predict.cu)."""
    sc = _scorer(3)  # n_sets 1,225 -> ld 1,536: three tile columns
    n_dec = 6
    buf = np.arange(sc.out_elems(n_dec), dtype=np.float64)
    v = sc.view_full(buf, n_dec)
    RC, T = sc.ld // 512, 512
    for d, k, o, r in [(0, 0, 0, 0), (5, 1, sc.E - 1, sc.ld - 1), (3, 1, 7, 600), (4, 0, 2, 1023)]:
        off = ((((d // 4) * sc.E + o) * RC + r // T) * 8 + (d % 4) * 2 + k) * T + r % T
        assert v[d, k, o, r] == buf[off]


def test_host_buffer_variant_equals_device_variant():
    sc = _scorer(3)
    C = _golden.load("candidates_golden.npz")
    W = np.stack([C["w"], C["w"] * 0.5])
    dev_out = sc.alloc(2)
    sc.score(torch.tensor(W, device="cuda").contiguous(), dev_out)
    host_out = np.empty(sc.out_elems(2), dtype=np.float32)
    scratch = torch.empty(sc.scratch_elems(2), dtype=torch.float32, device="cuda")
    sc.score_host(np.ascontiguousarray(W), host_out, scratch)
    torch.cuda.synchronize()
    # rows of the padded decisions (the tile holds 4) are never written: compare the logical arrays
    np.testing.assert_array_equal(sc.view_full(host_out, 2), sc.view_full(dev_out.cpu().numpy(), 2))


@pytest.mark.parametrize("fused", [True, False])
def test_pipelined_steps_equal_one_shot(fused):
    """pipeline_step (forward of step k overlapped with the feature build of
    step k+1 on a side stream) gives the one-shot results, for decision
    counts that are and are not multiples of the per-block chunk."""
    sc = _scorer(3)
    rng = np.random.default_rng(5)
    Ws = [rng.normal(0, 0.5, size=(n, 2, 7)) for n in (7, 4, 1, 9)]
    outs = [sc.alloc(len(W)) for W in Ws]
    sc.pipeline_start(fused=fused)
    for W, out in zip(Ws, outs):
        sc.pipeline_step(torch.tensor(W, device="cuda").contiguous(), out)
    sc.pipeline_join()
    for W, out in zip(Ws, outs):
        ref = sc.alloc(len(W))
        sc.score(torch.tensor(W, device="cuda").contiguous(), ref)
        np.testing.assert_array_equal(sc.view_full(out.cpu().numpy(), len(W)), sc.view_full(ref.cpu().numpy(), len(W)))


def test_best_candidate_step_equals_argmin_of_full_output():
    """intf_candidate_best_step (the per-decision reduction a scheduler
    consumes) equals the argmin of the materialised predictions of the same
    step: the same fp32 values, the lowest multiset rank on ties; the host
    variant equals the device step; and against the fp64 restatement the
    chosen candidate is the best one within the 1e-5 tolerance."""
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles
    from paper_2512_18725_b200.sweep import c2_decision_coefs

    sc = _scorer(4)
    W = np.ascontiguousarray(c2_decision_coefs(32, 0.5)[[0, 7, 19, 31]])
    coefs = torch.tensor(W, dtype=torch.float64, device="cuda").contiguous()
    out = sc.alloc(4)
    bufs = [sc.alloc_best(4) for _ in range(3)]
    sc.pipeline_start(fused=True)
    sc.pipeline_step(coefs, out)  # materialised step (features of step 0)
    sc.best_step(coefs, bufs[0], bufs[1])  # best step (features rebuilt by step 0's prep blocks)
    sc.pipeline_join()
    y = sc.view(out.cpu().numpy(), 4)
    val, rank = sc.decode_best(bufs[0], 4)
    am = y.argmin(axis=-1)
    assert np.array_equal(rank, am)
    assert np.array_equal(val, np.take_along_axis(y, am[..., None], -1)[..., 0])
    assert np.all(bufs[1].cpu().numpy() == -1)  # reset for the next step
    scratch = torch.empty(sc.best_scratch_elems(4), dtype=torch.float32, device="cuda")
    hb = np.zeros(4 * 2 * sc.E, dtype=np.uint64)
    sc.best_host(W, hb, scratch)
    torch.cuda.synchronize()
    assert np.array_equal(hb.view(np.int64), bufs[0].cpu().numpy())
    ta = gen_synthetic_profiles().arrays()
    ref = O.candidate_predictions_all(ta.solo, ta.thr, 4, W, 0.5)
    rmin = ref.min(axis=-1)
    np.testing.assert_allclose(val, rmin, rtol=RTOL, atol=0)
    np.testing.assert_allclose(np.take_along_axis(ref, rank[..., None], -1)[..., 0], rmin, rtol=2 * RTOL, atol=0)


def test_real_decisions_from_replayed_sweep():
    """The candidate set of every real decision of a replayed C5 sweep (the
    running set at each dispatch, `simcore.py:150-171`) against the heap-engine
    oracle's replay: the same running multiset for every batch; every own row
    scored against it equals the enumeration's prediction for that column
    (materialised by the C2 kernel), the best own row is its argmin, and the
    FIFO batch's prediction is its own entry."""
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles
    from paper_2512_18725_b200.sweep import c2_decision_coefs, c5_scenarios

    table = gen_synthetic_profiles()
    ta = table.arrays()
    specs = c5_scenarios(table, 64, start=300)
    pipe = engine.ReplayPipeline(specs, ta, scale=1.5)
    pipe.run()
    sc = engine.CandidateScorer(ta, cap=4, alpha=0.5)
    sc.prepare()
    W = c2_decision_coefs(32, 0.5)[-1]
    coefs = torch.tensor(W, dtype=torch.float64, device="cuda").contiguous()
    rank, own = sc.dispatch_decisions(pipe)
    best0, chosen0 = sc.score_decisions(coefs, rank, own)  # features read in the enumeration's layout
    sc.prepare_decisions()
    best, chosen = sc.score_decisions(coefs, rank, own)  # decision-major copy
    live = (rank >= 0).repeat_interleave(2)
    assert torch.equal(best, best0) and torch.equal(chosen[live], chosen0[live])
    assert torch.isnan(chosen[~live]).all()
    out = sc.alloc(1)
    sc.score(coefs.reshape(1, 2, 7).contiguous(), out)
    y = sc.view(out.cpu().numpy(), 1)[0]  # [2][E][n_sets]
    h = pipe.fetch()
    rank, own = rank.cpu().numpy(), own.cpu().numpy()
    bk = best.cpu().numpy().view(np.uint64).reshape(-1, 2)
    ch = chosen.cpu().numpy().reshape(-1, 2)
    otab = O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr)
    n_dec = 0
    for s, spec in enumerate(specs):
        v = pipe.scenario(h, s)
        ref = O.run_scenario(spec, otab)
        ro = pipe.pb.scen[s].req_off
        ids = [d["model_id"] for d in spec["deployed"]]
        rows = [ta.row(ids[m], int(z)) for m, z in zip(ref["b_model"], ref["b_size"])]
        for b in range(len(rows)):
            peers = [rows[c] for c in range(b) if ref["b_completion"][c] > ref["b_start"][b]]
            r = engine.multiset_rank(peers, sc.E, 4)
            assert rank[ro + b] == r and own[ro + b] == rows[b], (s, b)
            for k in range(2):
                col = y[k, :, r]
                key = int(bk[ro + b, k])
                hi = np.uint32(key >> 32)
                val = np.array([hi & np.uint32(0x7FFFFFFF) if hi >> np.uint32(31) else ~hi], dtype=np.uint32)
                assert val.view(np.float32)[0] == col.min() and (key & 0xFFFFFFFF) == int(col.argmin())
                assert ch[ro + b, k] == col[rows[b]]
            n_dec += 1
        assert np.all(rank[ro + len(rows): ro + pipe.pb.scen[s].req_cap] == -1)
    assert n_dec > 10000


def test_pipelined_host_best_calls_equal_single_calls():
    """intf_best_candidates_host_pipelined (each call scores from the features
    the previous call built and builds the next call's in the same launch)
    returns the same keys as the one-shot host call, call after call."""
    from paper_2512_18725_b200.sweep import c2_decision_coefs

    sc = _scorer(4)
    W = c2_decision_coefs(32, 0.5)
    scr1 = torch.empty(sc.best_scratch_elems(8), dtype=torch.float32, device="cuda")
    scr2 = torch.empty(sc.best_scratch_elems(8) + sc.ws_elems, dtype=torch.float32, device="cuda")
    for k in range(4):
        Wk = np.ascontiguousarray(W[8 * k: 8 * k + 8])
        a = np.zeros(2 * 8 * sc.E, dtype=np.uint64)
        b = np.zeros_like(a)
        sc.best_host(Wk, a, scr1)
        sc.best_host_pipelined(Wk, b, scr2)
        torch.cuda.synchronize()
        assert np.array_equal(a, b), k


def test_pipelined_host_best_pinned_one_launch():
    """With a pinned result buffer and <= 32 decisions the pipelined host call
    is ONE launch (coefficients as a kernel parameter, the last block writes
    the keys into the pinned buffer and re-arms them): the same keys as the
    one-shot call, call after call, with the decision count changing and with
    pageable (copy path) and pinned calls interleaved on the same scratch."""
    from paper_2512_18725_b200.sweep import c2_decision_coefs

    sc = _scorer(4)
    W = c2_decision_coefs(32, 0.5)
    scr1 = torch.empty(sc.best_scratch_elems(32), dtype=torch.float32, device="cuda")
    scr2 = torch.empty(sc.best_scratch_elems(32) + sc.ws_elems, dtype=torch.float32, device="cuda")
    pinned = torch.empty(2 * 32 * sc.E, dtype=torch.int64).pin_memory()
    plan = [(0, 32, True), (3, 11, True), (7, 32, True), (1, 5, False), (2, 8, True), (9, 23, True), (0, 32, False),
            (4, 32, True)]
    for k, (lo, hi, pin) in enumerate(plan):
        Wk = np.ascontiguousarray(W[lo:hi])
        n = hi - lo
        a = np.zeros(2 * n * sc.E, dtype=np.uint64)
        sc.best_host(Wk, a, scr1)
        b = pinned.numpy().view(np.uint64)[: 2 * n * sc.E] if pin else np.zeros_like(a)
        b[:] = 0
        sc.best_host_pipelined(Wk, b, scr2)
        torch.cuda.synchronize()
        assert np.array_equal(a, b), (k, lo, hi, pin)


def test_host_sync_call_equals_single_calls():
    """intf_best_candidates_host_sync returns with the keys in host memory
    (pinned: the kernel's completion word; pageable: a stream sync), equal to
    the one-shot call, for pinned and pageable buffers."""
    from paper_2512_18725_b200.sweep import c2_decision_coefs

    sc = _scorer(4)
    W = c2_decision_coefs(32, 0.5)
    scr1 = torch.empty(sc.best_scratch_elems(32), dtype=torch.float32, device="cuda")
    scr2 = torch.empty(sc.best_scratch_elems(32) + sc.ws_elems, dtype=torch.float32, device="cuda")
    pinned = torch.empty(2 * 32 * sc.E, dtype=torch.int64).pin_memory()
    for k, (lo, hi, pin) in enumerate([(0, 32, True), (5, 21, True), (2, 9, False), (0, 32, True), (8, 12, True)]):
        Wk = np.ascontiguousarray(W[lo:hi])
        a = np.zeros(2 * (hi - lo) * sc.E, dtype=np.uint64)
        sc.best_host(Wk, a, scr1)
        torch.cuda.synchronize()
        b = pinned.numpy().view(np.uint64)[: a.size] if pin else np.zeros_like(a)
        b[:] = 0
        sc.best_host_pipelined(Wk, b, scr2, sync=True)
        assert np.array_equal(a, b), (k, lo, hi, pin)  # no synchronisation: the call returned with the keys
