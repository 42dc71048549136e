"""Pin the CPU oracle (oracle/) to the reference's golden outputs before it
is trusted as the checker (tests/golden/make_golden.py ran the unmodified
reference).  CPU only."""
import math

import numpy as np
import pytest

import oracle as O
from tests import _golden


def _otab(name="default"):
    t = _golden.table(name)
    return O.TableArrays(t.models, t.max_bs, t.solo, t.thr)


@pytest.mark.parametrize("name", _golden.scenario_names())
def test_oracle_replay_bit_exact(name):
    spec = _golden.spec(name)
    tab = _otab(str(_golden.replay()[name + "/table"]))
    rep = O.run_scenario(spec, tab)
    assert rep["status"] == 0
    assert _golden.compare_replay(rep, name) == []
    G = _golden.replay()
    for mi, (ewma, alpha) in enumerate(_golden.MODES):
        X, y, _ = O.samples_from_replay(rep, spec, tab, bool(ewma), alpha)
        np.testing.assert_array_equal(X, G[f"{name}/x_mode{mi}"])
        np.testing.assert_array_equal(y, G[f"{name}/y_mode{mi}"])


def test_oracle_slo_report_matches_golden():
    G = _golden.replay()
    for name in ("bundled_seed7", "churn0_1", "c4slice", "rand13"):
        spec = _golden.spec(name)
        tab = _otab(str(G[name + "/table"]))
        rep = O.run_scenario(spec, tab)
        ids = [d["model_id"] for d in spec["deployed"]]
        models = [ids[m] for m in rep["arr_model"]]
        comp = rep["b_completion"][rep["r_batch"]]
        out = O.slo_report(models, rep["arr_t"], comp, rep["r_slo_met"])
        for j, m in enumerate(G[name + "/slo_models"]):
            n, sat, p50, p95, p99 = out[str(m)]
            assert n == G[name + "/slo_n"][j] and sat == G[name + "/slo_sat"][j]
            assert [p50, p95, p99] == list(G[name + "/slo_p"][j])
        warm = O.slo_report(models, rep["arr_t"], comp, rep["r_slo_met"], warmup_fraction=0.2)
        np.testing.assert_array_equal(np.array([list(warm[k]) for k in sorted(warm)]), G[name + "/slo_warm_p"])


def test_oracle_rng_known_answers():
    R = _golden.load("rng_golden.npz")
    keys = R["noise_keys"]
    got = np.array([O.noise_draw(int(s), int(b), int(k), 0.05) for s, b, k in keys])
    np.testing.assert_array_equal(got, R["noise_sigma005"])
    got2 = np.array([O.noise_draw(int(s), int(b), int(k), 0.02) for s, b, k in keys[:400]])
    np.testing.assert_array_equal(got2, R["noise_sigma002"])
    np.testing.assert_array_equal(O.random_doubles(O.int_words(*R["uniform_seed"]), 5000), R["uniform"])
    np.testing.assert_array_equal(O.standard_normals(O.int_words(*R["normal_seed"]), len(R["normal"])), R["normal"])
    np.testing.assert_array_equal([O.c_exp(float(x)) for x in R["exp_x"]], R["exp_y"])
    np.testing.assert_array_equal([O.c_log1p(float(x)) for x in R["log1p_x"]], R["log1p_y"])


def test_oracle_noise_sigma_zero_is_one():
    assert O.noise_draw(5, 3, 1, 0.0) == 1.0


def test_oracle_predictor_restatement_matches_golden():
    P = _golden.load("predict_golden.npz")
    for mi in range(4):
        X, y, cut = P[f"ewma/mode{mi}/X"], P[f"ewma/mode{mi}/y"], int(P[f"ewma/mode{mi}/ncut"])
        w, b = O.fit_ols_xy(X[:cut], y[:cut])
        np.testing.assert_array_equal(w, P[f"ewma/mode{mi}/w"])
        assert b == float(P[f"ewma/mode{mi}/b"])
        rep = O.eval_report([O.predict(w, b, x) for x in X[cut:]], y[cut:])
        np.testing.assert_array_equal(np.array(rep), P[f"ewma/mode{mi}/report"])
    for seed in (0, 1):
        p = f"drift{seed}/"
        w0, b0 = O.fit_ols_xy(P[p + "Xtrain"], P[p + "ytrain"])
        np.testing.assert_array_equal(w0, P[p + "w0"])
        np.testing.assert_array_equal(O.rls_init_P(P[p + "Xtrain"]), P[p + "P0"])
        for ts in ("TestSet1", "TestSet2", "TestSet3"):
            X, y = P[p + ts + "/X"], P[p + ts + "/y"]
            pr, w, b, _ = O.prequential(w0, b0, X, y, "sgd")
            np.testing.assert_array_equal(pr, P[p + ts + "/sgd_pred"])
            np.testing.assert_array_equal(np.append(w, b), P[p + ts + "/sgd_w"])
            pr, w, b, Pm = O.prequential(w0, b0, X, y, "rls", P=O.rls_init_P(P[p + "Xtrain"]))
            np.testing.assert_array_equal(pr, P[p + ts + "/rls_pred"])
            np.testing.assert_array_equal(Pm, P[p + ts + "/rls_P"])
    w, b = O.fit_ols_xy(P["ridge/X"], P["ridge/y"])
    np.testing.assert_array_equal(np.append(w, b), P["ridge/w"])


def test_oracle_fit_ols_ill_conditioned_matches_golden():
    """The oracle's fit_ols_xy on the rank-deficient / ill-conditioned designs
    of tests/golden/ols_rank_golden.npz (reference results)."""
    from tests.golden.ols_rank_designs import designs

    G = _golden.load("ols_rank_golden.npz")
    for name, (X, y) in designs().items():
        if len(y) > 10000:
            continue  # the 2*10^5-row design is for the device QR only (time)
        w, b = O.fit_ols_xy(X, y)
        np.testing.assert_array_equal(np.append(w, b), G[f"{name}/params"])


def test_oracle_candidates_match_golden():
    C = _golden.load("candidates_golden.npz")
    tab = _otab()
    for cap in (2, 3):
        own, peers = C[f"cap{cap}/own"], C[f"cap{cap}/peers"]
        for i in range(0, len(own), 7):
            pe = [q for q in peers[i] if q >= 0]
            yc, yf = O.candidate_predictions(int(own[i]), pe, tab.solo, tab.thr, C["w"][0], C["w"][1], 0.5)
            assert yc == C[f"cap{cap}/y_coarse"][i] and yf == C[f"cap{cap}/y_fine"][i]


# ---- known-answer tests carried over from the reference suite
def test_oracle_hand_example_slowdown():
    # `test_simcore.py:49-53`: own=colo=(0.6,0.5,0.4) -> excess (0.2,0,0) -> 1.2
    import ctypes

    L = O.lib()
    a = np.array([1.0, 1.5, 0.5])
    e = np.array([0.6 + 0.6 - 1.0, 0.0, 0.0])
    dot = L.oracle_ddot(a.ctypes.data_as(O.PD), e.ctypes.data_as(O.PD), 3)
    assert math.isclose(1.0 + dot, 1.2, rel_tol=1e-12)
    del ctypes


def test_oracle_ewma_hand_example():
    # `test_colocation.py:61-64`: EWMA(0.5) from (0.4,0.4,0.4) observing (0.8,0,0.4) -> (0.6,0.2,0.4)
    x = O.features(np.array([[0.4, 0.4, 0.4], [0.8, 0.0, 0.4]]), np.zeros(3), True, 0.5)
    np.testing.assert_allclose(x[3:], [0.6, 0.2, 0.4])


def test_oracle_sgd_hand_step():
    # `test_predict.py:115-121`: zero model, x=(1,0,...), y=10, eta=0.01 -> w0=0.1, b=0.1
    w, b = O.sgd_update(np.zeros(6), 0.0, np.array([1.0, 0, 0, 0, 0, 0]), 10.0, 0.01)
    assert math.isclose(w[0], 0.1) and math.isclose(b, 0.1)


def test_oracle_percentile_examples():
    # `test_metrics.py:26-31`
    assert O.percentile([1, 2, 3, 4], 50) == 2
    assert O.percentile([15, 20, 35, 40, 50], 40) == 20
    assert O.percentile([3, 1, 2], 100) == 3
    assert O.percentile([5], 0) == 5


@pytest.mark.parametrize("cap", [2, 3, 4])
def test_vectorised_candidate_restatement_matches_reference(cap):
    """`oracle.candidate_predictions_all` (the checker of the full C2
    enumeration on the GPU) against predictions the reference's own
    functions composed (cap 2 in full, cap 3/4 subsampled); the only
    difference allowed is the ddot's fma rounding (~1e-16)."""
    from paper_2512_18725_b200 import engine

    tab = _golden.table("default")
    C = _golden.load("candidates_golden.npz")
    Y = O.candidate_predictions_all(tab.solo, tab.thr, cap, C["w"][None], float(C["alpha"]))[0]
    own, peers = C[f"cap{cap}/own"], C[f"cap{cap}/peers"]
    M = O.multisets(len(tab.solo), cap)
    idx = np.array([engine.multiset_rank([q for q in pe if q >= 0], len(tab.solo), cap) for pe in peers])
    for i, pe in zip(idx, peers):
        assert list(M[i][M[i] >= 0]) == sorted(q for q in pe if q >= 0)
    np.testing.assert_allclose(Y[0, own, idx], C[f"cap{cap}/y_coarse"], rtol=1e-14, atol=0)
    np.testing.assert_allclose(Y[1, own, idx], C[f"cap{cap}/y_fine"], rtol=1e-14, atol=0)
    # and the scalar restatement's features bit for bit on a sample
    Xs, Xf = O.candidate_features_all(tab.solo, tab.thr, cap, float(C["alpha"]))
    for o, pe, i in list(zip(own, peers, idx))[::37]:
        hist = O.candidate_history(int(o), [q for q in pe if q >= 0], tab.solo, tab.thr)
        assert np.array_equal(Xs[o, i], O.features(hist, tab.thr[o], False, 1.0))
        assert np.array_equal(Xf[o, i], O.features(hist, tab.thr[o], True, float(C["alpha"])))


def test_oracle_scenario_eval_matches_reference():
    """`oracle.scenario_eval` (the C5 coarse / fine / adaptive evaluation
    checker) against the reference's own split_samples / fit_ols / rls_init /
    evaluate on the first 24 sweep scenarios (tests/golden/c5eval_golden.npz)."""
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles
    from paper_2512_18725_b200.sweep import c5_scenario

    G = _golden.load("c5eval_golden.npz")
    table = gen_synthetic_profiles()
    otab = _otab("default")
    for i in G["idx"]:
        spec = c5_scenario(table, int(i))
        got = O.scenario_eval(O.run_scenario(spec, otab), spec, otab)
        ref = G["reports"][i]
        if np.isnan(ref[0, 0]):
            assert got is None
            continue
        np.testing.assert_allclose(got, ref, rtol=1e-9, err_msg=f"scenario {i}")


def test_oracle_drift_experiment_matches_reference():
    """`oracle.drift_experiment` (the C3 CPU baseline and checker) against the
    reference's drift_experiment cells for seeds 0 and 1."""
    from paper_2512_18725_b200 import experiments as ex
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles

    P = _golden.load("predict_golden.npz")
    table = gen_synthetic_profiles()
    otab = _otab("default")
    for seed in (0, 1):
        cells = O.drift_experiment(ex.drift_specs(ex.default_drift_base(table, seed)), otab)
        assert [f"{d}/{m}" for d, m, _, _ in cells] == [str(k) for k in P[f"drift{seed}/cell_keys"]]
        np.testing.assert_allclose([[c[2], c[3]] for c in cells], P[f"drift{seed}/cells"], rtol=1e-9)
