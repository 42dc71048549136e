"""The interactive step API (`simcore.py:103-208`, `GpuState`) on B200: the
reference's known-answer cases (`pkg/tests/test_simcore.py:46-140`) restated,
its spy tests (`test_simcore.py:259-277`, `test_acceptance.py:90-140`) run
through `run_scenario`, and a GpuState driven along the device's formation
trace equal to the reference goldens bit for bit on every golden scenario."""
import numpy as np
import pytest

from tests import _golden

pytestmark = pytest.mark.gpu


def _profile_table(ta):
    import paper_2512_18725_b200 as p

    entries = {}
    for mi, m in enumerate(ta.models):
        for bs in range(1, ta.max_bs + 1):
            r = mi * ta.max_bs + bs - 1
            entries[(m, bs)] = p.ModelProfile(m, bs, float(ta.solo[r]), *(float(v) for v in ta.thr[r]))
    return p.ProfileTable(entries, ta.max_bs)


def _three():
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200.profiles import Archetype

    return p.gen_synthetic_profiles([Archetype("alpha", 10.0, 1.0, (0.60, 0.50, 0.40)),
                                     Archetype("bravo", 10.0, 1.0, (0.60, 0.50, 0.40)),
                                     Archetype("charlie", 4.0, 1.0, (0.30, 0.20, 0.10))])


def _batch(bid, model, size=1, t=0.0):
    from paper_2512_18725_b200.batcher import BatchRequest
    from paper_2512_18725_b200.workload import RequestEvent

    return BatchRequest(bid, model, tuple(RequestEvent(bid * 100 + i, model, t, t + 1e9) for i in range(size)), t)


NOISELESS_SIGMA = 0.0


def _state(cap):
    import paper_2512_18725_b200 as p

    return p.GpuState(concurrency_cap=cap, oracle=p.InterferenceOracle(noise_sigma=NOISELESS_SIGMA))


def test_hand_example_and_solo():
    import paper_2512_18725_b200 as p

    o = p.InterferenceOracle(noise_sigma=0.0)
    assert p.oracle_slowdown((0.9, 0.9, 0.9), (0.0, 0.0, 0.0), o) == 1.0
    assert p.oracle_slowdown((0.6, 0.5, 0.4), (0.6, 0.5, 0.4), o) == pytest.approx(1.2)
    with pytest.raises(ValueError):
        p.oracle_slowdown((-0.1, 0.5, 0.5), (0.0, 0.0, 0.0), o)
    table = _three()
    st = _state(2)
    st.dispatch(_batch(0, "alpha"), table)
    t, kind, key, payload = st.advance_to_next_event()
    assert (t, kind, key) == (pytest.approx(10.0), 0, 0)
    out = st.complete(payload[0])
    assert out.interference_ratio == pytest.approx(1.0) and out.n_segments == 1


def test_piecewise_reprojection_by_hand():
    """alpha alone for 4 ms, then bravo joins: alpha's completion is
    re-projected to 4 + 6 * slowdown and its work integrates to 10."""
    import paper_2512_18725_b200 as p

    table = _three()
    slow = p.oracle_slowdown(table.get("alpha", 1).throughputs(), table.get("bravo", 1).throughputs(),
                             p.InterferenceOracle(noise_sigma=0.0))
    assert slow > 1.0
    st = _state(2)
    a = st.dispatch(_batch(0, "alpha"), table)
    st.now_ms = 4.0
    a.close_segment(4.0)
    st._reseat(a)
    st.dispatch(_batch(1, "bravo"), table)
    assert a.current_slowdown == pytest.approx(slow)
    expected = 4.0 + (10.0 - 4.0) * slow
    live = [e for e in sorted(st.events) if e[4][0] is a and e[4][1] == a.completion_gen]
    assert live and live[0][0] == pytest.approx(expected)
    st.now_ms = expected
    a.close_segment(expected)
    assert a.progress_ms == pytest.approx(10.0)


def test_cap_and_past_event_errors():
    import paper_2512_18725_b200 as p

    table = _three()
    st = _state(2)
    st.dispatch(_batch(0, "alpha"), table)
    st.dispatch(_batch(1, "bravo"), table)
    assert not st.can_dispatch()
    with pytest.raises(p.SimulationError):
        st.dispatch(_batch(2, "alpha"), table)
    st2 = _state(1)
    st2.now_ms = 10.0
    with pytest.raises(p.SimulationError):
        st2.push_event(9.0, 2, 0, None)


def test_noisy_reseat_uses_device_noise():
    """With noise, a hand-driven reseat draws default_rng([seed, batch, seg])
    lognormal on the device: equal to the noise-table draw of the replay."""
    import paper_2512_18725_b200 as p

    o = p.InterferenceOracle(noise_sigma=0.1, seed=5)
    assert o.noise_draw(3, 1) == o.noise_draw(3, 1) != o.noise_draw(3, 2)
    st = p.GpuState(2, o)
    table = _three()
    rb = st.dispatch(_batch(3, "charlie"), table)
    assert rb.segments[0].slowdown == o.noise_draw(3, 0)  # alone: (1 + 0) * noise


def _scenario(table, models, rate, seed=0, cap=2, duration_s=2.0, window_ms=1.0, sigma=0.0):
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200.workload import default_slo_ms

    dep = tuple(p.DeployedModel(m, rate, slo_ms=default_slo_ms(table, m, factor=100.0)) for m in models)
    return p.ScenarioSpec(deployed=dep, duration_s=duration_s, batching_window_ms=window_ms, concurrency_cap=cap,
                          seed=seed, oracle=p.InterferenceOracle(noise_sigma=sigma, seed=seed))


def test_spy_running_never_exceeds_cap():
    """`test_simcore.py:259-277`: a wrapped GpuState.dispatch sees every
    dispatch of run_scenario (the device replay plus the step-API walk along
    its trace), the running set never above the cap and reaching it."""
    import paper_2512_18725_b200 as p

    table = _three()
    observed = []
    original = p.GpuState.dispatch

    def spying_dispatch(self, batch, tbl):
        rb = original(self, batch, tbl)
        observed.append(len(self.running))
        assert len(self.running) <= self.concurrency_cap
        return rb

    p.GpuState.dispatch = spying_dispatch
    try:
        res = p.run_scenario(_scenario(table, ["alpha", "bravo"], rate=120.0, seed=8, cap=2, duration_s=1.0), table)
    finally:
        p.GpuState.dispatch = original
    assert max(observed) == 2 and len(observed) == len(res.outcomes)


def test_spy_criterion_3_conservation():
    """`test_acceptance.py:90-140`: 100 random noiseless scenarios, work
    conservation, cap-1 exactness, and the cap observed at every dispatch."""
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200.workload import default_slo_ms

    table = p.gen_synthetic_profiles()
    models = table.models()
    rng = np.random.default_rng(42)
    observed = []
    original = p.GpuState.dispatch

    def spying_dispatch(self, batch, tbl):
        rb = original(self, batch, tbl)
        observed.append((len(self.running), self.concurrency_cap))
        return rb

    p.GpuState.dispatch = spying_dispatch
    try:
        for i in range(100):
            cap = int(rng.integers(1, 4))
            chosen = list(rng.choice(models, size=rng.integers(1, 4), replace=False))
            dep = tuple(p.DeployedModel(m, float(rng.uniform(20.0, 150.0)),
                                        slo_ms=default_slo_ms(table, m, factor=100.0)) for m in chosen)
            spec = p.ScenarioSpec(deployed=dep, duration_s=float(rng.uniform(0.3, 1.0)),
                                  batching_window_ms=float(rng.uniform(0.0, 5.0)), concurrency_cap=cap,
                                  seed=int(rng.integers(0, 10_000)), oracle=p.InterferenceOracle(noise_sigma=0.0),
                                  name=f"rand{i}")
            for out in p.run_scenario(spec, table).outcomes:
                integrated = sum((s.t_end - s.t_begin) / s.slowdown for s in out.segments)
                assert abs(integrated - out.profiled_ms) <= 1e-6 * out.profiled_ms
                if cap == 1:
                    assert out.interference_ratio == 1.0
    finally:
        p.GpuState.dispatch = original
    assert observed and all(1 <= r <= c for r, c in observed)
    assert any(r == c and c > 1 for r, c in observed)


def test_step_walk_equals_goldens():
    """A GpuState driven along the device's formation trace reproduces the
    reference's outcomes and segments bit for bit (noise on, every golden
    scenario of the bundled table and the 16-model slice)."""
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.simcore import _drive_step_api
    from paper_2512_18725_b200.workload import scenario_from_dict

    G = _golden.replay()
    for tname in ("default", "t16"):
        if tname not in _golden.table_names():
            continue
        ta = _golden.table(tname)
        table = _profile_table(ta)
        names = _golden.scenario_names(tname)
        pipe, h = engine.run_batch([_golden.spec(n) for n in names], ta)
        for s, n in enumerate(names):
            spec = scenario_from_dict(_golden.spec(n))
            outs = _drive_step_api(spec, table, pipe.scenario(h, s))
            p = n + "/"
            assert [o.batch_id for o in outs] == list(G[p + "o_batch"]), n
            assert np.array_equal([o.start_ms for o in outs], G[p + "o_start"]), n
            assert np.array_equal([o.measured_duration_ms for o in outs], G[p + "o_measured"]), n
            assert np.array_equal([o.completion_time_ms for o in outs], G[p + "o_completion"]), n
            segs = [sg for o in outs for sg in o.segments]
            assert np.array_equal([sg.t_begin for sg in segs], G[p + "s_tbegin"]), n
            assert np.array_equal([sg.t_end for sg in segs], G[p + "s_tend"]), n
            assert np.array_equal([sg.slowdown for sg in segs], G[p + "s_slowdown"]), n
            assert np.array_equal(np.array([sg.colo for sg in segs]).reshape(-1, 3), G[p + "s_colo"]), n
