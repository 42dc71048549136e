"""The SLO report's percentile selection (k_slo: radix digits over the
scenario's key range, first histogram shared by the quantiles, bins of <= 32
records ranked by one warp; k_slo_big for long traces) on crafted arrivals
that stress its edges, against the reference's slo_report (`metrics.py:49-79`,
restated in oracle.slo_report) on the oracle's replay of the same arrivals:

* bursts of 40 simultaneous requests batched together (40 equal latencies:
  a selected bin above the warp-rank limit, resolved by further passes),
* the same beyond the shared-memory key cache (> 2,048 requests),
* latencies spanning many binades (an overloaded cap-1 burst),
* one and two requests,
* warm-up cutoffs at half the span and at the last arrival (`metrics.py:60-67`)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _spec(table, models, name, max_bs=64, window=2.0, cap=2, sigma=0.05, seed=0):
    dep = [{"model_id": m, "arrival_rate_rps": 100.0, "slo_ms": 20.0 * table.get(m, 1).solo_duration_ms}
           for m in models]
    return {"name": name, "duration_s": 1.0, "batching_window_ms": window, "max_batch_size": max_bs,
            "concurrency_cap": cap, "seed": seed, "colocation_mode": "static", "ewma_alpha": 1.0,
            "oracle": {"beta_l2": 1.0, "beta_dram": 1.5, "beta_sm": 0.5, "noise_sigma": sigma, "seed": seed},
            "deployed": dep}


def _arrivals(parts):
    """parts: [(times, model)] -> time-sorted (t, model) (stable: model order on ties)."""
    t = np.concatenate([np.asarray(p[0], dtype=np.float64) for p in parts])
    m = np.concatenate([np.full(len(p[0]), p[1], dtype=np.int32) for p in parts])
    o = np.lexsort((m, t))
    return t[o], m[o]


def _cases(table):
    models = table.models()
    rng = np.random.default_rng(11)
    bursts = np.repeat(np.arange(0.0, 1000.0, 50.0), 40)  # 20 bursts x 40 simultaneous requests
    sparse = np.sort(rng.uniform(0.0, 1000.0, 120))
    big = np.repeat(np.arange(0.0, 1000.0, 14.0), 35)  # 72 bursts x 35: > 2,048 requests
    over = np.sort(rng.uniform(0.0, 1.0, 600))  # 600 requests in 1 ms, cap 1: queueing over many binades
    late = np.sort(rng.uniform(0.0, 1000.0, 300))
    return [
        (_spec(table, models[:2], "ties"), _arrivals([(bursts, 0), (sparse, 1)])),
        (_spec(table, models[2:4], "ties_uncached", cap=3), _arrivals([(big, 0), (sparse, 1)])),
        (_spec(table, models[4:6], "binades", cap=1, window=0.0, max_bs=4), _arrivals([(over, 0), (late, 1)])),
        (_spec(table, models[:1], "one"), _arrivals([(np.array([3.0]), 0)])),
        (_spec(table, models[:2], "two"), _arrivals([(np.array([3.0]), 0), (np.array([3.0]), 1)])),
    ]


def _check(specs, arrivals, ta, warmup_fraction=0.0):
    from paper_2512_18725_b200 import engine

    pipe, h = engine.run_batch(specs, ta, arrivals=arrivals, warmup_fraction=warmup_fraction)
    otab = O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr)
    max_tie = 0
    for s, (spec, arr) in enumerate(zip(specs, arrivals)):
        v = pipe.scenario(h, s)
        ref = O.run_scenario(spec, otab, arrivals=arr)
        assert v["status"] == 0 and ref["status"] == 0, spec["name"]
        assert np.array_equal(v["b_completion"], ref["b_completion"]), spec["name"]
        ids = [d["model_id"] for d in spec["deployed"]]
        lat = ref["b_completion"][ref["r_batch"]] - ref["arr_t"]
        rep = O.slo_report([ids[m] for m in ref["arr_model"]], ref["arr_t"], lat + ref["arr_t"], ref["r_slo_met"],
                           warmup_fraction)
        for m, mid in enumerate(ids):
            if mid not in rep:
                assert v["slo_n"][m] == 0, (spec["name"], mid)
                continue
            n, sat, p50, p95, p99 = rep[mid]
            assert v["slo_n"][m] == n and v["slo_met"][m] / n == sat, (spec["name"], mid)
            assert list(v["slo_p"][m]) == [p50, p95, p99], (spec["name"], mid, list(v["slo_p"][m]), (p50, p95, p99))
            _, counts = np.unique(lat[ref["arr_model"] == m], return_counts=True)
            max_tie = max(max_tie, int(counts.max()))
    return max_tie


def test_slo_edges_vs_reference():
    from paper_2512_18725_b200.sweep import table16

    t16, _ = table16()
    cases = _cases(t16)
    max_tie = _check([c[0] for c in cases], [c[1] for c in cases], t16.arrays())
    assert max_tie > 32  # the tie case really exceeds the warp-rank limit


def test_slo_edges_warmup_cutoffs():
    from paper_2512_18725_b200.sweep import table16

    t16, _ = table16()
    cases = _cases(t16)
    _check([c[0] for c in cases], [c[1] for c in cases], t16.arrays(), warmup_fraction=0.5)
    # fraction 1.0: the cutoff is the last arrival, only the latest records stay
    _check([c[0] for c in cases[:3]], [c[1] for c in cases[:3]], t16.arrays(), warmup_fraction=1.0)


def test_long_list_burst_batches_bucket_fallback():
    """Caller-supplied arrivals on lists past the long-list threshold (chunked
    formation, time-bucket batch merge): bursts of 5,000 simultaneous requests
    form 78 max-size batches at one instant -- a time bucket far above 64
    batches, ranked by the binary-search fallback -- and the replay equals the
    oracle's (batches, outcomes, records, SLO report)."""
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.sweep import table16

    t16, _ = table16()
    ta = t16.arrays()
    models = t16.models()
    burst = np.repeat([10.0, 400.0, 800.0], 5000)
    rng = np.random.default_rng(5)
    other = np.sort(rng.uniform(0.0, 1000.0, 4500))
    spec = _spec(t16, models[:2], "long_bursts", max_bs=64, window=5.0, cap=3)
    arr = _arrivals([(burst, 0), (other, 1)])
    pipe, h = engine.run_batch([spec], ta, arrivals=[arr])
    v = pipe.scenario(h, 0)
    otab = O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr)
    ref = O.run_scenario(spec, otab, arrivals=arr)
    assert v["status"] == 0 and ref["status"] == 0
    for k in ("order", "b_model", "b_size", "b_formed", "b_start", "b_completion", "b_measured", "r_batch",
              "r_slo_met"):
        assert np.array_equal(np.asarray(v[k]), np.asarray(ref[k])), k
    _, counts = np.unique(np.asarray(ref["b_formed"]), return_counts=True)
    assert counts.max() > 64  # the fallback really ran
