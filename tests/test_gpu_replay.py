"""GPU parity: the sm_100a replay pipeline (arrivals -> replay -> SLO ->
features) against the reference's golden outputs, bit-exact."""
import numpy as np
import pytest

from tests import _golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu_runs():
    from paper_2512_18725_b200 import _abi, engine

    runs = {}
    for tname in _golden.table_names():
        names = _golden.scenario_names(tname)
        preds = [_abi.Predictor(ewma=e, alpha=a, w=(0.1, -0.2, 0.3, 0.05, 0.4, -0.1, 1.0)) for e, a in _golden.MODES]
        pipe, h = engine.run_batch([_golden.spec(n) for n in names], _golden.table(tname), preds=preds)
        runs[tname] = (names, pipe, h)
    return runs


def _views(gpu_runs):
    for tname, (names, pipe, h) in gpu_runs.items():
        for s, n in enumerate(names):
            yield n, pipe.scenario(h, s)


def test_replay_bit_exact_all_golden_scenarios(gpu_runs):
    bad = {}
    for name, v in _views(gpu_runs):
        assert v["status"] == 0, (name, v["status"])
        fails = _golden.compare_replay(v, name)
        if fails:
            bad[name] = fails
    assert not bad, bad


def test_features_bit_exact(gpu_runs):
    G = _golden.replay()
    for name, v in _views(gpu_runs):
        for mi in range(4):
            np.testing.assert_array_equal(v["X"][mi], G[f"{name}/x_mode{mi}"], err_msg=f"{name} mode{mi}")
        np.testing.assert_array_equal(v["Y"], G[f"{name}/y_mode0"], err_msg=name)


def test_predictions_match_fma_chain(gpu_runs):
    w = np.array([0.1, -0.2, 0.3, 0.05, 0.4, -0.1])
    for name, v in _views(gpu_runs):
        for mi in range(4):
            ref = v["X"][mi] @ w + 1.0
            np.testing.assert_allclose(v["Yhat"][mi], ref, rtol=1e-12, atol=0)


def test_slo_report_matches_reference(gpu_runs):
    G = _golden.replay()
    for tname, (names, pipe, h) in gpu_runs.items():
        for s, name in enumerate(names):
            v = pipe.scenario(h, s)
            ids = list(G[f"{name}/slo_models"])
            spec = _golden.spec(name)
            dep = [d["model_id"] for d in spec["deployed"]]
            for j, mid in enumerate(ids):
                m = dep.index(mid)
                assert v["slo_n"][m] == G[f"{name}/slo_n"][j]
                assert v["slo_met"][m] / v["slo_n"][m] == G[f"{name}/slo_sat"][j]
                np.testing.assert_array_equal(v["slo_p"][m], G[f"{name}/slo_p"][j], err_msg=f"{name} {mid}")


def test_dispatch_trace_matches_oracle_and_cap(gpu_runs):
    """Running-set size at every dispatch (the spy of `test_acceptance.py:98-106`,
    `test_simcore.py:259-277`): equal to the heap-engine oracle's, never above cap."""
    import oracle as O

    for name, v in _views(gpu_runs):
        spec = _golden.spec(name)
        t = _golden.table(str(_golden.replay()[name + "/table"]))
        ref = O.run_scenario(spec, O.TableArrays(t.models, t.max_bs, t.solo, t.thr))
        assert np.array_equal(v["b_running"], ref["b_running"]), name
        if len(v["b_running"]):
            assert 1 <= v["b_running"].min() and v["b_running"].max() <= spec["concurrency_cap"]


def test_reseat_and_segment_counts_match_oracle(gpu_runs):
    """Event-level shortcuts in the warp replay (cap-1 chain, bulk formations
    while full, the completion reseat a same-instant dispatch pops) must keep
    the reference's reseat count (`simcore.py:133-141`, every `_reseat` call,
    3,590 for the bundled seed-7 trace) and kept-segment count."""
    import oracle as O

    for tname, (names, pipe, h) in gpu_runs.items():
        tab = _golden.table(tname)
        otab = O.TableArrays(tab.models, tab.max_bs, tab.solo, tab.thr)
        for s, n in enumerate(names):
            v = pipe.scenario(h, s)
            ref = O.run_scenario(_golden.spec(n), otab)
            assert (v["n_reseats"], v["n_segments"]) == (ref["n_reseats"], ref["n_segments"]), n
    v = dict(_views(gpu_runs))["bundled_seed7"]
    assert v["n_reseats"] == 3590 and v["n_segments"] == 3200
