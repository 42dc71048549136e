"""Busy-period sharding: the segmented replay (speculative idle
boundaries, verified and merged) is bit-identical to the serial replay and to
the reference goldens, also when most speculative boundaries fail."""
import numpy as np
import pytest

from tests import _golden

pytestmark = pytest.mark.gpu


def _run(specs, table, **kw):
    from paper_2512_18725_b200 import engine

    pipe = engine.ReplayPipeline(specs, table, scale=1.5)
    stats = engine.replay_segmented(pipe, **kw)
    return pipe, pipe.fetch(), stats


@pytest.mark.parametrize("slow,min_len", [(2.0, 64), (0.0, 1), (0.5, 4)])
def test_segmented_replay_matches_goldens(slow, min_len):
    for tname in _golden.table_names():
        names = _golden.scenario_names(tname)
        pipe, h, stats = _run([_golden.spec(n) for n in names], _golden.table(tname), slow=slow, min_len=min_len)
        for s, n in enumerate(names):
            v = pipe.scenario(h, s)
            assert v["status"] == 0, n
            assert _golden.compare_replay(v, n) == [], (n, stats)
        assert stats["jobs_final"] <= stats["jobs_initial"]


@pytest.mark.parametrize("slow,min_len,passes", [(2.0, 16, 0), (0.5, 4, 0), (0.0, 1, 0), (2.0, 64, 4), (2.0, 64, 1),
                                                 (0.5, 4, -3)])
def test_long_trace_segmented_equals_serial(slow, min_len, passes):
    """A 2x10^5-request trace (req_cap >= 32768: block-parallel plan/verify,
    long-list arrivals) replayed as busy-period jobs -- also with most
    speculative boundaries failing (slow 0.5 / 0.0: long runs of merges) --
    equals the whole-trace replay and the CPU oracle.  passes > 0: passes
    queued with device-side job counts (1: too few, the host loop finishes);
    passes < 0: the same, deferred (finish() after the queued SLO)."""
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.sweep import c4_scenario, table16

    t16, arch = table16()
    spec = c4_scenario(t16, arch, n_requests=2e5)
    ta = t16.arrays()
    if passes >= 0:
        pipe, h, stats = _run([spec], ta, slow=slow, min_len=min_len, passes=passes)
        assert stats["jobs_final"] > 10, stats  # the trace really was replayed in parallel pieces
        if min_len <= 4:  # more jobs than one 6,144-job verify tile (k_jobs_verify_big's tile loop)
            assert stats["jobs_initial"] > 6144, stats
    else:
        pipe = engine.ReplayPipeline([spec], ta, scale=1.5)
        fin = engine.replay_segmented(pipe, slow=slow, min_len=min_len, passes=-passes, stats=False)
        fin()
        h = pipe.fetch()
    ser, hs = engine.run_batch([spec], ta)
    a, b = pipe.scenario(h, 0), ser.scenario(hs, 0)
    assert a["status"] == 0 and b["status"] == 0
    for k in ("order", "b_model", "b_size", "b_start", "b_completion", "b_measured", "b_nseg", "r_batch",
              "r_slo_met"):
        assert np.array_equal(a[k], b[k]), k
    ia = np.concatenate([np.arange(o, o + n) for o, n in zip(a["b_seg_off"], a["b_nseg"])])
    ib = np.concatenate([np.arange(o, o + n) for o, n in zip(b["b_seg_off"], b["b_nseg"])])
    for k in ("s_tbegin", "s_tend", "s_slowdown"):
        assert np.array_equal(a[k][ia], b[k][ib]), k
    assert np.array_equal(a["slo_p"], b["slo_p"]) and a["n_reseats"] == b["n_reseats"]
    # against the CPU oracle (heap engine); the SLO report takes the grid-wide path here
    import oracle as O

    ref = O.run_scenario(spec, O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr))
    assert np.array_equal(a["order"], ref["order"]) and np.array_equal(a["b_completion"], ref["b_completion"])
    assert np.array_equal(a["r_slo_met"], ref["r_slo_met"])
    ids = [d["model_id"] for d in spec["deployed"]]
    rep = O.slo_report([ids[m] for m in ref["arr_model"]], ref["arr_t"], ref["b_completion"][ref["r_batch"]],
                       ref["r_slo_met"])
    for m, mid in enumerate(ids):
        n, sat, p50, p95, p99 = rep[mid]
        assert a["slo_n"][m] == n and a["slo_met"][m] / a["slo_n"][m] == sat
        assert list(a["slo_p"][m]) == [p50, p95, p99]


def test_sweep_segmented_equals_whole_scenario_jobs():
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.sweep import c5_scenarios

    table = p.gen_synthetic_profiles()
    specs = c5_scenarios(table, 256)
    ta = table.arrays()
    a_pipe = engine.ReplayPipeline(specs, ta, scale=1.5)
    stats = engine.replay_segmented(a_pipe, min_len=8)
    ha = a_pipe.fetch()
    b_pipe = engine.ReplayPipeline(specs, ta, scale=1.5)
    b_pipe.run()
    hb = b_pipe.fetch()
    assert stats["jobs_final"] > len(specs)
    for s in range(len(specs)):
        a, b = a_pipe.scenario(ha, s), b_pipe.scenario(hb, s)
        assert a["status"] == 0 and b["status"] == 0
        for k in ("order", "b_start", "b_completion", "b_measured", "b_nseg", "r_slo_met", "slo_p", "slo_met"):
            assert np.array_equal(a[k], b[k]), (s, k)
        assert a["n_reseats"] == b["n_reseats"]


def test_two_long_traces_in_one_batch():
    """Two long traces + short scenarios in one batch: per-scenario regions of
    the block-parallel plan/verify scratch do not collide."""
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.sweep import c4_scenario, table16

    t16, arch = table16()
    specs = [c4_scenario(t16, arch, n_requests=1e5, seed=5), _golden.spec("c4slice"),
             c4_scenario(t16, arch, n_requests=1.2e5, seed=6)]
    ta = t16.arrays()
    pipe, h, stats = _run(specs, ta, slow=1.0, min_len=8)
    ser, hs = engine.run_batch(specs, ta)
    for s in range(3):
        a, b = pipe.scenario(h, s), ser.scenario(hs, s)
        assert a["status"] == 0 and b["status"] == 0
        for k in ("order", "b_start", "b_completion", "b_measured", "b_nseg", "r_slo_met"):
            assert np.array_equal(a[k], b[k]), (s, k)
        assert a["n_reseats"] == b["n_reseats"] and a["n_segments"] == b["n_segments"]


def test_device_and_host_planned_sharding_agree():
    from paper_2512_18725_b200 import engine

    names = _golden.scenario_names("default")
    specs = [_golden.spec(n) for n in names]
    a = engine.ReplayPipeline(specs, _golden.table("default"), scale=1.5)
    engine.replay_segmented(a, slow=0.5, min_len=4)
    b = engine.ReplayPipeline(specs, _golden.table("default"), scale=1.5)
    engine.replay_segmented_host(b, slow=0.5, min_len=4)
    ha, hb = a.fetch(), b.fetch()
    for s, n in enumerate(names):
        va, vb = a.scenario(ha, s), b.scenario(hb, s)
        assert _golden.compare_replay(va, n) == [] and _golden.compare_replay(vb, n) == []
        assert va["n_reseats"] == vb["n_reseats"] and va["n_segments"] == vb["n_segments"]
