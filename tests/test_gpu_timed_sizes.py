"""Parity at the sizes bench.py times (VERDICT r1 "weak #1"):

* C2: the full cap-4 enumeration (999,600 candidates x coarse/fine) for
  several of the bench's refit decisions, through the bench's kernel
  (k_cand_step, pipelined), against the vectorised restatement
  `oracle.candidate_predictions_all` -- itself pinned to the reference's own
  functions on cap 2/3/4 subsamples (tests/test_oracle_golden.py);
* C5: all 10^4 bench scenarios (default_rng([2512, i]), LPT order, the bench's
  three predictors) bit-exact against the heap-engine oracle;
* C4: the 10^6-request bench trace, busy-period sharded as in the bench,
  bit-exact against the oracle, including the grid-wide SLO report;
* the warm-up-trimmed slo_report on the device (`metrics.py:60-64`).
"""
import numpy as np
import pytest
import torch

import oracle as O
from tests import _golden

pytestmark = pytest.mark.gpu
RTOL = 1e-5  # north star: predictions within 1e-5 relative in fp32


def _otab(ta):
    return O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr)


# ---------------------------------------------------------------- C2
@pytest.fixture(scope="module")
def c2_setup():
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles
    from paper_2512_18725_b200.sweep import c2_decision_coefs

    ta = gen_synthetic_profiles().arrays()
    W = c2_decision_coefs(32, 0.5)
    sc = engine.CandidateScorer(ta, cap=4, alpha=0.5)
    return ta, W, sc


def test_c2_cap4_full_enumeration_bench_decisions(c2_setup):
    """Every one of the 999,600 cap-4 candidates, both predictors, for 4 of the
    bench's 32 refit decisions, produced by the bench's pipelined k_cand_step:
    relative error <= 1e-5 against the fp64 restatement, no absolute floor
    (the OLS-fitted predictors give interference ratios ~1, far from 0)."""
    ta, W, sc = c2_setup
    dsel = [0, 10, 21, 31]
    Wd = np.ascontiguousarray(W[dsel])
    coefs = torch.tensor(Wd, dtype=torch.float64, device="cuda").contiguous()
    outs = [sc.alloc(len(dsel)), sc.alloc(len(dsel))]
    sc.pipeline_start(fused=True)
    for k in range(3):  # step 0 uses the warm-up features, steps 1-2 the features built by the previous step
        sc.pipeline_step(coefs, outs[k & 1])
    sc.pipeline_join()
    y = sc.view(outs[0].cpu().numpy(), len(dsel)).astype(np.float64)
    ref = O.candidate_predictions_all(ta.solo, ta.thr, 4, Wd, 0.5)
    assert y.shape == ref.shape == (len(dsel), 2, 48, 20825)
    rel = np.abs(y - ref) / np.abs(ref)
    assert np.abs(ref).min() > 0.1, np.abs(ref).min()
    assert rel.max() <= RTOL, (rel.max(), np.unravel_index(rel.argmax(), rel.shape))
    y1 = sc.view(outs[1].cpu().numpy(), len(dsel))
    assert np.array_equal(y1, sc.view(outs[0].cpu().numpy(), len(dsel)))


def test_c2_cap4_full_enumeration_random_coefficients(c2_setup):
    """Random N(0, 0.5) coefficients can cancel to |y| ~ 0, where a relative
    bound is meaningless for ANY fp32 forward.  The stated bound there is the
    fp32 forward's own error model: |dy| <= 1e-5 |y| + 2^-20 (sum_i |w_i x_i| + |b|)
    (2^-20 ~ 8 fp32 ulps of the dot's magnitude), checked on every candidate."""
    ta, _, sc = c2_setup
    W = np.random.default_rng(11).normal(0, 0.5, size=(2, 2, 7))
    coefs = torch.tensor(W, dtype=torch.float64, device="cuda").contiguous()
    out = sc.alloc(2)
    sc.score(coefs, out)
    y = sc.view(out.cpu().numpy(), 2).astype(np.float64)
    Xs, Xf = O.candidate_features_all(ta.solo, ta.thr, 4, 0.5)
    for d in range(2):
        for k, X in enumerate((Xs, Xf)):
            ref = X @ W[d, k, :6] + W[d, k, 6]
            mag = np.abs(X) @ np.abs(W[d, k, :6]) + abs(W[d, k, 6])
            bound = RTOL * np.abs(ref) + 2.0 ** -20 * mag
            assert np.all(np.abs(y[d, k] - ref) <= bound), (d, k, np.max(np.abs(y[d, k] - ref) / bound))


# ---------------------------------------------------------------- C5
@pytest.fixture(scope="module")
def c5_run():
    from paper_2512_18725_b200 import _abi, engine
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles
    from paper_2512_18725_b200.sweep import c2_decision_coefs, c5_scenarios, lpt_order

    table = gen_synthetic_profiles()
    ta = table.arrays()
    W = c2_decision_coefs(32, 0.5)
    preds = [_abi.Predictor(ewma=0, alpha=1.0, w=tuple(W[-1, 0])), _abi.Predictor(ewma=1, alpha=0.5, w=tuple(W[-1, 1])),
             _abi.Predictor(ewma=1, alpha=0.5, w=tuple(W[0, 1]))]
    specs = lpt_order(c5_scenarios(table, 10000))
    pipe = engine.ReplayPipeline(specs, ta, preds=preds, scale=1.5)  # the bench's construction
    pipe.run()
    pipe.run()  # a second sweep on the same buffers (the bench re-runs pipelines)
    return specs, ta, W, pipe, pipe.fetch()


def test_c5_sweep_all_bench_scenarios_bit_exact(c5_run):
    specs, ta, W, pipe, h = c5_run
    otab = _otab(ta)
    bad = {}
    for s, spec in enumerate(specs):
        v = pipe.scenario(h, s)
        ref = O.run_scenario(spec, otab)
        assert v["status"] == 0 and ref["status"] == 0, (s, v["status"], ref["status"])
        fails = [k for k in ("order", "b_model", "b_size", "b_formed", "b_start", "b_completion", "b_measured",
                             "b_nseg", "b_running", "arr_t", "arr_model", "r_batch", "r_slo_met")
                 if not np.array_equal(v[k], ref[k])]
        if not fails:
            ia = _golden.outcome_segment_index(v["b_seg_off"], v["b_nseg"], v["order"])
            ib = _golden.outcome_segment_index(ref["b_seg_off"], ref["b_nseg"], ref["order"])
            fails += [k for k in ("s_tbegin", "s_tend", "s_slowdown", "s_colo") if not np.array_equal(v[k][ia], ref[k][ib])]
            if (v["n_reseats"], v["n_segments"]) != (ref["n_reseats"], ref["n_segments"]):
                fails.append("counts")
            ids = [d["model_id"] for d in spec["deployed"]]
            rep = O.slo_report([ids[m] for m in ref["arr_model"]], ref["arr_t"], ref["b_completion"][ref["r_batch"]],
                               ref["r_slo_met"])
            for m, mid in enumerate(ids):
                if mid not in rep:
                    fails += ["slo_n"] if v["slo_n"][m] != 0 else []
                    continue
                n, sat, p50, p95, p99 = rep[mid]
                if v["slo_n"][m] != n or v["slo_met"][m] / n != sat or list(v["slo_p"][m]) != [p50, p95, p99]:
                    fails.append(f"slo:{mid}")
        if fails:
            bad[s] = fails
            if len(bad) > 10:
                break
    assert not bad, bad


def test_c5_sweep_features_and_predictions(c5_run):
    """Features and fp64 predictions of the bench's three predictors on every
    10th scenario (plus the 64 heaviest), bit-exact features, predictions
    equal to the fma-chain ddot (`predict.py:43-44`)."""
    specs, ta, W, pipe, h = c5_run
    otab = _otab(ta)
    modes = [(False, 1.0, W[-1, 0]), (True, 0.5, W[-1, 1]), (True, 0.5, W[0, 1])]
    for s in sorted(set(range(0, len(specs), 10)) | set(range(64))):
        v = pipe.scenario(h, s)
        ref = O.run_scenario(specs[s], otab)
        for mi, (e, a, w) in enumerate(modes):
            X, y, _ = O.samples_from_replay(ref, specs[s], otab, e, a)
            assert np.array_equal(v["X"][mi], X), (s, mi)
            assert np.array_equal(v["Y"], y), s
            np.testing.assert_allclose(v["Yhat"][mi], X @ w[:6] + w[6], rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- C4
def test_c4_bench_trace_bit_exact():
    """The bench's 10^6-request C4 trace (seed 1, 16 models, bs <= 64, cap 4),
    replayed as busy-period jobs with the bench's 4 queued passes, against the
    heap-engine oracle: every batch, segment, request record and the grid-wide
    SLO report."""
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.sweep import c4_scenario, table16

    t16, arch = table16()
    spec = c4_scenario(t16, arch, n_requests=1e6, seed=1)
    ta = t16.arrays()
    pipe = engine.ReplayPipeline([spec], ta, scale=1.2)
    stats = engine.replay_segmented(pipe, passes=4)
    v = pipe.scenario(pipe.fetch(), 0)
    ref = O.run_scenario(spec, _otab(ta))
    assert v["status"] == 0 and ref["status"] == 0
    assert len(v["arr_t"]) > 990000 and stats["jobs_final"] > 1000, stats
    for k in ("arr_t", "arr_model", "order", "b_model", "b_size", "b_formed", "b_start", "b_completion", "b_measured",
              "b_nseg", "r_batch", "r_slo_met"):
        assert np.array_equal(v[k], ref[k]), k
    ia = _golden.outcome_segment_index(v["b_seg_off"], v["b_nseg"], v["order"])
    ib = _golden.outcome_segment_index(ref["b_seg_off"], ref["b_nseg"], ref["order"])
    for k in ("s_tbegin", "s_tend", "s_slowdown", "s_colo"):
        assert np.array_equal(v[k][ia], ref[k][ib]), k
    assert (v["n_reseats"], v["n_segments"]) == (ref["n_reseats"], ref["n_segments"])
    ids = [d["model_id"] for d in spec["deployed"]]
    rep = O.slo_report([ids[m] for m in ref["arr_model"]], ref["arr_t"], ref["b_completion"][ref["r_batch"]],
                       ref["r_slo_met"])
    for m, mid in enumerate(ids):
        n, sat, p50, p95, p99 = rep[mid]
        assert v["slo_n"][m] == n and v["slo_met"][m] / n == sat
        assert list(v["slo_p"][m]) == [p50, p95, p99], mid


# ---------------------------------------------------------------- warm-up SLO
def _check_warm(v, spec, warm_rows, name):
    """warm_rows: sorted-by-model rows (n, satisfaction, p50, p95, p99) of the
    reference's slo_report(records, warmup_fraction=0.2); models with no
    request after the cutoff are absent there and have n = 0 here."""
    ids = [d["model_id"] for d in spec["deployed"]]
    present = sorted({ids[m] for m in range(len(ids)) if v["slo_n"][m] > 0})
    assert len(present) == len(warm_rows), name
    for mid, row in zip(present, warm_rows):
        m = ids.index(mid)
        n, sat, p50, p95, p99 = row
        assert v["slo_n"][m] == n and v["slo_met"][m] / v["slo_n"][m] == sat, (name, mid)
        assert list(v["slo_p"][m]) == [p50, p95, p99], (name, mid)


def test_warmup_slo_report_matches_reference_goldens():
    """run_batch(warmup_fraction=0.2) -> the device cutoff path of k_slo
    against the reference's slo_report(records, warmup_fraction=0.2)
    (`metrics.py:60-64`) frozen in the goldens, for every golden scenario."""
    from paper_2512_18725_b200 import engine

    G = _golden.replay()
    for tname in _golden.table_names():
        names = _golden.scenario_names(tname)
        specs = [_golden.spec(n) for n in names]
        pipe, h = engine.run_batch(specs, _golden.table(tname), warmup_fraction=0.2)
        for s, n in enumerate(names):
            v = pipe.scenario(h, s)
            if len(v["arr_t"]) == 0:
                continue
            _check_warm(v, specs[s], G[n + "/slo_warm_p"], n)


def test_warmup_slo_report_long_trace_grid_path():
    """The same cutoff through the grid-wide k_slo_big_* passes (a 2x10^5
    request trace), against the oracle's slo_report with the warm-up trim."""
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.sweep import c4_scenario, table16

    t16, arch = table16()
    spec = c4_scenario(t16, arch, n_requests=2e5)
    ta = t16.arrays()
    pipe, h = engine.run_batch([spec], ta, warmup_fraction=0.2)
    v = pipe.scenario(h, 0)
    ref = O.run_scenario(spec, _otab(ta))
    ids = [d["model_id"] for d in spec["deployed"]]
    rep = O.slo_report([ids[m] for m in ref["arr_model"]], ref["arr_t"], ref["b_completion"][ref["r_batch"]],
                       ref["r_slo_met"], warmup_fraction=0.2)
    _check_warm(v, spec, [rep[k] for k in sorted(rep)], "c4 2e5")
