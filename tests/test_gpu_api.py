"""The drop-in API (`import paper_2512_18725_b200 as intfsim`) returns the
reference's objects with bit-identical values (goldens)."""
import numpy as np
import pytest

from tests import _golden

pytestmark = pytest.mark.gpu


def _spec(name):
    from paper_2512_18725_b200.workload import scenario_from_dict

    return scenario_from_dict(_golden.spec(name))


def test_run_scenario_objects_bit_exact():
    import paper_2512_18725_b200 as p

    G = _golden.replay()
    table = p.gen_synthetic_profiles()
    for name in ("bundled_seed7", "churn0_2", "rand7"):
        res = p.run_scenario(_spec(name), table)
        assert [o.batch_id for o in res.outcomes] == list(G[name + "/o_batch"])
        assert [o.completion_time_ms for o in res.outcomes] == list(G[name + "/o_completion"])
        assert [o.measured_duration_ms for o in res.outcomes] == list(G[name + "/o_measured"])
        segs = [s for o in res.outcomes for s in o.segments]
        assert [s.slowdown for s in segs] == list(G[name + "/s_slowdown"])
        assert [r.batch_id for r in res.records] == list(G[name + "/r_batch"])
        assert [r.slo_met for r in res.records] == [bool(v) for v in G[name + "/r_slo"]]
        mi = 0 if res.outcomes and _spec(name).colocation_mode.kind == "static" else 2
        np.testing.assert_array_equal(np.array([s.x for s in res.samples]).reshape(-1, 6), G[f"{name}/x_mode{mi}"])
        rep = p.slo_report(res.records)
        for j, m in enumerate(G[name + "/slo_models"]):
            r = rep[str(m)]
            assert (r.n_requests, r.slo_satisfaction) == (G[name + "/slo_n"][j], G[name + "/slo_sat"][j])
            assert [r.p50_latency_ms, r.p95_latency_ms, r.p99_latency_ms] == list(G[name + "/slo_p"][j])


def test_generate_arrivals_bit_exact():
    import paper_2512_18725_b200 as p

    G = _golden.replay()
    for name in ("bundled_seed0", "c4slice"):
        ev = p.generate_arrivals(_spec(name))
        assert [e.arrival_time_ms for e in ev] == list(G[name + "/arr_t"])


def test_samples_from_arbitrary_outcomes_and_estimators():
    import paper_2512_18725_b200 as p

    table = p.gen_synthetic_profiles()
    res = p.run_scenario(_spec("churn0_0"), table)
    plain = list(res.outcomes)  # drop the fast-path arrays: rebuild from objects
    for mode in (p.STATIC_MODE, p.ewma_mode(0.5)):
        a = p.samples_from_outcomes(plain, table, mode)
        b = p.samples_from_outcomes(res.outcomes, table, mode)
        np.testing.assert_array_equal([s.x for s in a], [s.x for s in b])
    est = p.init_estimate(0, p.ewma_mode(0.5), (0.4, 0.4, 0.4))
    p.observe(est, (0.8, 0.0, 0.4))
    np.testing.assert_allclose(est.r_hat, [0.6, 0.2, 0.4])


def test_percentile_examples():
    import paper_2512_18725_b200 as p

    assert p.percentile([1, 2, 3, 4], 50) == 2
    assert p.percentile([15, 20, 35, 40, 50], 40) == 20
    assert p.percentile([3, 1, 2], 100) == 3
    with pytest.raises(ValueError):
        p.percentile([], 50)


def test_empty_trace_and_edge_shapes():
    import paper_2512_18725_b200 as p

    table = p.gen_synthetic_profiles()
    spec = p.ScenarioSpec(deployed=(p.DeployedModel("resnet50", 0.0, 10.0),), duration_s=1.0)
    res = p.run_scenario(spec, table)
    assert res.outcomes == [] and res.records == []
    one = p.ScenarioSpec(deployed=(p.DeployedModel("resnet50", 500.0, 10.0),), duration_s=0.5,
                         batching_window_ms=0.0, max_batch_size=1, concurrency_cap=1,
                         oracle=p.InterferenceOracle(noise_sigma=0.0))
    res = p.run_scenario(one, table)
    assert res.outcomes and all(o.interference_ratio == 1.0 for o in res.outcomes)  # cap 1, sigma 0 (`test_acceptance.py:137-138`)


@pytest.mark.parametrize("n_requests,seed,dur", [(2e5, 3, None), (3e5, 17, None), (1.2e5, 5, 7.3), (6e4, 9, 0.05)])
def test_long_stream_arrivals_bit_exact_vs_oracle(n_requests, seed, dur):
    """Model streams of >= 4096 requests take the long-list path (every gap in
    parallel, k_gen_gaps; the cumulative sum as exact integer runs per binade,
    k_scan_binade, with real fp64 adds at binade crossings and ties):
    bit-exact against the oracle's sequential generator, incl. the
    overflow/retry path (scale 1.0 first) and a zero-rate model; durations
    from 50 ms (every stream inside a few binades, dense gaps) to ~1 h."""
    import oracle as O
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.sweep import c4_scenario, table16

    t16, arch = table16()
    spec = c4_scenario(t16, arch, n_requests=n_requests, seed=seed)
    if dur is not None:  # same rates' shape, another horizon (rates scaled to keep the request count)
        k = spec["duration_s"] / dur
        spec["duration_s"] = dur
        for d in spec["deployed"]:
            d["arrival_rate_rps"] *= k
    spec["deployed"][5]["arrival_rate_rps"] = 0.0
    ta = t16.arrays()
    (at, am), = engine.arrivals([spec], ta)
    ot, om = O.generate_arrivals(spec, O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr))
    assert len(at) > 0.75 * n_requests
    np.testing.assert_array_equal(at, ot)
    np.testing.assert_array_equal(am, om)


def test_long_stream_overflow_is_flagged_then_retried():
    """A long-list capacity below the stream length must raise the overflow
    status (k_fill_gaps: every draw below the horizon), and the retrying
    caller (engine.arrivals grows the capacity) still gets the exact stream."""
    import ctypes

    from paper_2512_18725_b200 import _abi, engine
    from paper_2512_18725_b200.sweep import c4_scenario, table16

    t16, arch = table16()
    spec = c4_scenario(t16, arch, n_requests=1e5, seed=4)
    ta = t16.arrays()
    pipe = engine.ReplayPipeline([spec], ta, scale=0.6, seg_stride=1)
    _abi.check(_abi.load().intf_generate_arrivals(ctypes.byref(pipe.batch), ctypes.byref(pipe.B),
                                                  engine.stream_ptr()), "arrivals")
    assert pipe.status()[0] & _abi.ST_OVERFLOW
    import oracle as O

    (at, am), = engine.arrivals([spec], ta)
    ot, om = O.generate_arrivals(spec, O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr))
    np.testing.assert_array_equal(at, ot)
    np.testing.assert_array_equal(am, om)
