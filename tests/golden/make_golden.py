"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED
reference (`/root/reference/pkg/src/intfsim`) in this container.

The reference cannot travel to the GPU box, so its outputs are frozen here as
compressed numpy archives; the parity tests (CPU and GPU) compare against
these files and never import the reference at run time.

    python tests/golden/make_golden.py          # rewrites tests/golden/*.npz
    python tests/golden/make_golden.py --candidates | --c5eval   # one fixture only

Contents
  replay_golden.npz   per scenario: spec JSON, profile table, arrivals,
                      outcomes (+segments), records, samples for 4 feature
                      modes, slo_report          (`simcore.py:218-310`,
                      `colocation.py:95-105`, `metrics.py:49-79`)
  predict_golden.npz  OLS fits / offline + prequential SGD/RLS evaluations on
                      the drift family and the EWMA experiment
                      (`predict.py:53-205`, `experiments.py:63-205`)
  rng_golden.npz      numpy/glibc known answers: noise draws, uniform and
                      normal streams, exp/log1p samples (`oracle.py:24-33`)
  c5eval_golden.npz   per-scenario coarse / fine / adaptive EvalReports of
                      the first C5 sweep scenarios (`experiments.py:44-60`,
                      `predict.py:53-205`)
  candidates_golden.npz  candidate-set predictions composed from reference
                      functions (colo sums `simcore.py:126-131`,
                      `estimate_from_history`, `finalize_features`, `predict`)
"""
from __future__ import annotations

import json
import math
import os
import sys
from dataclasses import replace

import numpy as np

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import intfsim  # noqa: E402
from intfsim import experiments as ex  # noqa: E402
from intfsim import predict as pr  # noqa: E402
from intfsim.colocation import STATIC_MODE, ewma_mode, estimate_from_history, finalize_features  # noqa: E402
from intfsim.metrics import slo_report  # noqa: E402
from intfsim.profiles import Archetype, DEFAULT_ARCHETYPES, gen_synthetic_profiles, load_profiles  # noqa: E402
from intfsim.workload import (  # noqa: E402
    DeployedModel,
    ScenarioSpec,
    default_slo_ms,
    drift_scenarios,
    load_scenario,
    rate_for_utilization,
    scenario_to_dict,
)
from intfsim.oracle import InterferenceOracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
MODES = [STATIC_MODE, ewma_mode(1.0 / 3.0), ewma_mode(0.5), ewma_mode(2.0 / 3.0)]


def table16():
    """C4 table: 6 default archetypes + 10 from default_rng(123), bs 1..64
    (SURVEY.md §8d)."""
    rng = np.random.default_rng(123)
    arch = list(DEFAULT_ARCHETYPES)
    for i in range(10):
        base = float(rng.uniform(0.8, 8.0))
        eff = float(rng.uniform(0.2, 0.95))
        mix = tuple(float(v) for v in rng.uniform(0.2, 0.6, size=3))
        arch.append(Archetype(f"synth_{i:02d}", base, eff, mix))
    return gen_synthetic_profiles(arch, seed=0, max_batch_size=64), arch


def table32():
    """32 models (6 default + 26 from default_rng(321)), bs 1..16: the widest
    deployment the kernels support (one lane per model)."""
    rng = np.random.default_rng(321)
    arch = list(DEFAULT_ARCHETYPES)
    for i in range(26):
        arch.append(Archetype(f"wide_{i:02d}", float(rng.uniform(0.8, 6.0)), float(rng.uniform(0.2, 0.95)),
                              tuple(float(v) for v in rng.uniform(0.1, 0.5, size=3))))
    return gen_synthetic_profiles(arch, seed=0, max_batch_size=16), arch


def table_arrays(table):
    models = table.models()
    mbs = table.max_batch_size
    solo = np.zeros(len(models) * mbs)
    thr = np.zeros((len(models) * mbs, 3))
    for mi, m in enumerate(models):
        for bs in range(1, mbs + 1):
            p = table.get(m, bs)
            solo[mi * mbs + bs - 1] = p.solo_duration_ms
            thr[mi * mbs + bs - 1] = p.throughputs()
    return models, mbs, solo, thr


def scenario_list(table, t16):
    out = []
    bundled = load_scenario("/root/reference/pkg/scenarios/mixed_three_model.json", table)
    for seed in (0, 7):
        out.append((f"bundled_seed{seed}", replace(bundled, seed=seed), "default"))
    for i, s in enumerate(ex.high_churn_suite(table, 0)):
        out.append((f"churn0_{i}", s, "default"))
    fam = drift_scenarios(ex.default_drift_base(table, 0))
    for name, s in fam.named():
        out.append((f"drift0_{name}", replace(s, colocation_mode=ewma_mode(0.5)), "default"))
    for cap in (1, 2, 3):
        out.append(
            (f"stress_cap{cap}", ex.symmetric_stress_scenario(table, ["resnet50", "yolov8n"], 1.1, 3, cap), "default")
        )
    # random scenarios in the style of test_acceptance.py:90-144 (noise on and off)
    rng = np.random.default_rng(4242)
    models = table.models()
    for i in range(16):
        cap = int(rng.integers(1, 5))
        chosen = list(rng.choice(models, size=int(rng.integers(1, 5)), replace=False))
        deployed = tuple(
            DeployedModel(m, float(rng.uniform(20.0, 400.0)), slo_ms=default_slo_ms(table, m, factor=float(rng.uniform(3, 30))))
            for m in chosen
        )
        sigma = 0.0 if i % 4 == 0 else float(rng.choice([0.02, 0.05, 0.1]))
        spec = ScenarioSpec(
            deployed=deployed,
            duration_s=float(rng.uniform(0.3, 1.5)),
            batching_window_ms=0.0 if i % 5 == 0 else float(rng.uniform(0.0, 8.0)),
            max_batch_size=int(rng.choice([1, 4, 8])),
            concurrency_cap=cap,
            seed=int(rng.integers(0, 2**40)) if i % 3 == 0 else int(rng.integers(0, 10000)),
            oracle=InterferenceOracle(noise_sigma=sigma, seed=int(rng.integers(0, 2**33))),
            name=f"rand{i}",
        )
        out.append((f"rand{i}", spec, "default"))
    # C4-shaped slice: 16 models, bs <= 64, cap 4 (short, so the fixture stays small)
    _, arch = t16
    dep = []
    rng = np.random.default_rng(99)
    for a in arch:
        dep.append(DeployedModel(a.model_id, rate_for_utilization(t16[0], a.model_id, float(rng.uniform(0.02, 0.08)), 64),
                                 slo_ms=20 * t16[0].get(a.model_id, 1).solo_duration_ms))
    out.append(
        (
            "c4slice",
            ScenarioSpec(deployed=tuple(dep), duration_s=0.25, batching_window_ms=12.0, max_batch_size=64,
                         concurrency_cap=4, seed=1, oracle=InterferenceOracle(noise_sigma=0.05, seed=1), name="c4slice"),
            "t16",
        )
    )
    # edge shapes: widest cap, 32 deployed models, zero-rate models, sigma 0, near-empty traces
    models = table.models()
    out.append(("edge_cap8", ScenarioSpec(
        deployed=tuple(DeployedModel(m, 150.0, default_slo_ms(table, m, 10.0)) for m in models), duration_s=0.8,
        batching_window_ms=3.0, concurrency_cap=8, seed=11, oracle=InterferenceOracle(noise_sigma=0.05, seed=3),
        name="edge_cap8"), "default"))
    out.append(("edge_zero_rate", ScenarioSpec(
        deployed=(DeployedModel("resnet50", 0.0, 10.0), DeployedModel("vgg19", 220.0, 40.0),
                  DeployedModel("yolov8n", 0.0, 5.0), DeployedModel("vit_b16", 90.0, 30.0)), duration_s=1.0,
        batching_window_ms=2.5, concurrency_cap=3, seed=5, oracle=InterferenceOracle(noise_sigma=0.1, seed=9),
        name="edge_zero_rate"), "default"))
    out.append(("edge_sigma0_cap4", ScenarioSpec(
        deployed=tuple(DeployedModel(m, 120.0, default_slo_ms(table, m, 8.0)) for m in models[:4]), duration_s=1.0,
        batching_window_ms=1.0, concurrency_cap=4, seed=2, oracle=InterferenceOracle(noise_sigma=0.0, seed=0),
        name="edge_sigma0_cap4"), "default"))
    out.append(("edge_tiny", ScenarioSpec(
        deployed=(DeployedModel("roberta_b", 400.0, 30.0), DeployedModel("convnext_b", 300.0, 35.0)),
        duration_s=0.004, batching_window_ms=0.5, concurrency_cap=2, seed=77, name="edge_tiny"), "default"))
    t32, arch32 = table32()
    out.append(("edge_wide32", ScenarioSpec(
        deployed=tuple(DeployedModel(a.model_id, 40.0, 25 * t32.get(a.model_id, 1).solo_duration_ms) for a in arch32),
        duration_s=0.6, batching_window_ms=6.0, max_batch_size=16, concurrency_cap=8, seed=21,
        oracle=InterferenceOracle(noise_sigma=0.05, seed=2**40 + 7), name="edge_wide32"), "t32"))
    return out


def replay_golden(table, t16):
    tabs = {"default": table, "t16": t16[0], "t32": table32()[0]}
    arrs = {}
    names = []
    for name, spec, tname in scenario_list(table, t16):
        tab = tabs[tname]
        res = intfsim.run_scenario(spec, tab)
        arrivals = intfsim.generate_arrivals(spec)
        dep_idx = {d.model_id: i for i, d in enumerate(spec.deployed)}
        p = name + "/"
        names.append(name)
        arrs[p + "spec"] = np.array(json.dumps(scenario_to_dict(spec)))
        arrs[p + "table"] = np.array(tname)
        arrs[p + "arr_t"] = np.array([a.arrival_time_ms for a in arrivals])
        arrs[p + "arr_model"] = np.array([dep_idx[a.model_id] for a in arrivals], dtype=np.int32)
        oc = res.outcomes
        arrs[p + "o_batch"] = np.array([o.batch_id for o in oc], dtype=np.int64)
        arrs[p + "o_model"] = np.array([dep_idx[o.model_id] for o in oc], dtype=np.int32)
        arrs[p + "o_size"] = np.array([o.batch_size for o in oc], dtype=np.int32)
        arrs[p + "o_start"] = np.array([o.start_ms for o in oc])
        arrs[p + "o_measured"] = np.array([o.measured_duration_ms for o in oc])
        arrs[p + "o_profiled"] = np.array([o.profiled_ms for o in oc])
        arrs[p + "o_completion"] = np.array([o.completion_time_ms for o in oc])
        arrs[p + "o_nseg"] = np.array([o.n_segments for o in oc], dtype=np.int32)
        segs = [s for o in oc for s in o.segments]
        arrs[p + "s_tbegin"] = np.array([s.t_begin for s in segs])
        arrs[p + "s_tend"] = np.array([s.t_end for s in segs])
        arrs[p + "s_slowdown"] = np.array([s.slowdown for s in segs])
        arrs[p + "s_colo"] = np.array([s.colo for s in segs]).reshape(-1, 3)
        rec = res.records
        arrs[p + "r_batch"] = np.array([r.batch_id for r in rec], dtype=np.int64)
        arrs[p + "r_dispatch"] = np.array([r.dispatch_ms for r in rec])
        arrs[p + "r_completion"] = np.array([r.completion_ms for r in rec])
        arrs[p + "r_slo"] = np.array([r.slo_met for r in rec], dtype=np.uint8)
        for mi, mode in enumerate(MODES):
            sm = intfsim.colocation.samples_from_outcomes(oc, tab, mode, scenario=spec.name)
            arrs[p + f"x_mode{mi}"] = np.array([s.x for s in sm]).reshape(-1, 6)
            arrs[p + f"y_mode{mi}"] = np.array([s.y for s in sm])
        rep = slo_report(rec)
        ids = sorted(rep)
        arrs[p + "slo_models"] = np.array(ids)
        arrs[p + "slo_n"] = np.array([rep[m].n_requests for m in ids])
        arrs[p + "slo_sat"] = np.array([rep[m].slo_satisfaction for m in ids])
        arrs[p + "slo_p"] = np.array([[rep[m].p50_latency_ms, rep[m].p95_latency_ms, rep[m].p99_latency_ms] for m in ids])
        rep2 = slo_report(rec, warmup_fraction=0.2)
        arrs[p + "slo_warm_p"] = np.array(
            [[rep2[m].n_requests, rep2[m].slo_satisfaction, rep2[m].p50_latency_ms, rep2[m].p95_latency_ms, rep2[m].p99_latency_ms] for m in sorted(rep2)]
        )
        print(f"{name:22s} req={len(rec):6d} batches={len(oc):5d} segs={len(segs):6d}")
    for tname, tab in tabs.items():
        models, mbs, solo, thr = table_arrays(tab)
        arrs[f"_table/{tname}/models"] = np.array(models)
        arrs[f"_table/{tname}/max_bs"] = np.array(mbs)
        arrs[f"_table/{tname}/solo"] = solo
        arrs[f"_table/{tname}/thr"] = thr
    arrs["_names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "replay_golden.npz"), **arrs)


def predict_golden(table):
    arrs = {}
    # ewma_experiment on the seed-0 churn suite (`experiments.py:63-89`)
    suite = ex.high_churn_suite(table, 0)
    results = [intfsim.run_scenario(s, table) for s in suite]
    for mi, mode in enumerate(MODES):
        samples = []
        for spec, res in zip(suite, results):
            samples += intfsim.colocation.samples_from_outcomes(res.outcomes, table, mode, scenario=spec.name)
        train, test = ex.split_samples(samples)
        m = pr.fit_ols(train)
        rep = pr.evaluate(m, test)
        arrs[f"ewma/mode{mi}/X"] = np.array([s.x for s in samples])
        arrs[f"ewma/mode{mi}/y"] = np.array([s.y for s in samples])
        arrs[f"ewma/mode{mi}/ncut"] = np.array(len(train))
        arrs[f"ewma/mode{mi}/w"] = m.w
        arrs[f"ewma/mode{mi}/b"] = np.array(m.b)
        arrs[f"ewma/mode{mi}/report"] = np.array([rep.mse, rep.rel_p25, rep.rel_p50, rep.rel_p75, rep.rel_p95, rep.n_samples])
    # drift_experiment internals (`experiments.py:153-205`), seeds 0 and 1
    for seed in (0, 1):
        base = ex.default_drift_base(table, seed)
        fam = drift_scenarios(base)
        data = {}
        for name, spec in fam.named():
            spec = replace(spec, colocation_mode=ewma_mode(0.5))
            smp = intfsim.run_scenario(spec, table).samples
            if name != "TrainingSet":
                smp = smp[:300]
            data[name] = smp
        train = data["TrainingSet"]
        model0 = pr.fit_ols(train)
        Xtr = np.array([s.x for s in train])
        p = f"drift{seed}/"
        arrs[p + "Xtrain"] = Xtr
        arrs[p + "ytrain"] = np.array([s.y for s in train])
        arrs[p + "w0"] = model0.w
        arrs[p + "b0"] = np.array(model0.b)
        rls0 = pr.rls_init(model0, lam=0.99, X_train=Xtr)
        arrs[p + "P0"] = rls0.P
        for name in ("TestSet1", "TestSet2", "TestSet3"):
            smp = data[name]
            arrs[p + name + "/X"] = np.array([s.x for s in smp])
            arrs[p + name + "/y"] = np.array([s.y for s in smp])
            sgd = pr.SgdState(model0.copy(), eta=0.01)
            sgd_pred = [pr.score_and_update(sgd, s) for s in smp]
            rls = pr.rls_init(model0, lam=0.99, X_train=Xtr)
            rls_pred = [pr.score_and_update(rls, s) for s in smp]
            arrs[p + name + "/sgd_pred"] = np.array(sgd_pred)
            arrs[p + name + "/sgd_w"] = np.append(sgd.model.w, sgd.model.b)
            arrs[p + name + "/rls_pred"] = np.array(rls_pred)
            arrs[p + name + "/rls_w"] = np.append(rls.model.w, rls.model.b)
            arrs[p + name + "/rls_P"] = rls.P
        cells = ex.drift_experiment(base, table)
        arrs[p + "cells"] = np.array([[c.mse, c.n_samples] for c in cells])
        arrs[p + "cell_keys"] = np.array([f"{c.dataset}/{c.method}" for c in cells])
    # rank-deficient fit -> ridge fallback (`predict.py:58-61`)
    Xd = np.zeros((40, 6))
    Xd[:, :3] = np.random.default_rng(3).uniform(0.2, 0.6, size=(40, 3))
    yd = 1.0 + Xd[:, 0] * 0.3
    md = pr.fit_ols_xy(Xd, yd)
    arrs["ridge/X"] = Xd
    arrs["ridge/y"] = yd
    arrs["ridge/w"] = np.append(md.w, md.b)
    np.savez_compressed(os.path.join(HERE, "predict_golden.npz"), **arrs)


def rng_golden():
    arrs = {}
    rng = np.random.default_rng(11)
    seeds = rng.integers(0, 2**40, size=40)
    keys = []
    vals = []
    for s in list(seeds) + [0, 1, 7]:
        for b in (0, 1, 5, 1527, 99999, 2**32 + 3):
            for k in (0, 1, 2, 5, 19):
                keys.append((int(s), b, k))
                vals.append(float(np.random.default_rng([int(s), b, k]).lognormal(0.0, 0.05)))
    arrs["noise_keys"] = np.array(keys, dtype=np.uint64)
    arrs["noise_sigma005"] = np.array(vals)
    arrs["noise_sigma002"] = np.array([float(np.random.default_rng(list(k)).lognormal(0.0, 0.02)) for k in keys[:400]])
    arrs["uniform_seed"] = np.array([7, 2591491051], dtype=np.uint64)
    arrs["uniform"] = np.random.default_rng([7, 2591491051]).random(5000)
    arrs["normal_seed"] = np.array([5, 6, 7], dtype=np.uint64)
    arrs["normal"] = np.random.default_rng([5, 6, 7]).standard_normal(50000)
    xs = np.concatenate([rng.uniform(-8, 1, 20000), rng.standard_normal(20000) * 0.05])
    arrs["exp_x"] = xs
    arrs["exp_y"] = np.array([math.exp(v) for v in xs])
    us = np.concatenate([-rng.random(20000), rng.uniform(-0.999, 3, 20000)])
    arrs["log1p_x"] = us
    arrs["log1p_y"] = np.array([math.log1p(v) for v in us])
    np.savez_compressed(os.path.join(HERE, "rng_golden.npz"), **arrs)


def candidates_golden(table):
    """C2 candidate predictions via reference functions."""
    import itertools

    models, mbs, solo, thr = table_arrays(table)
    E = len(solo)
    suite = ex.high_churn_suite(table, 0)
    results = [intfsim.run_scenario(s, table) for s in suite]
    fits = []
    for mode in (STATIC_MODE, ewma_mode(0.5)):
        smp = []
        for spec, res in zip(suite, results):
            smp += intfsim.colocation.samples_from_outcomes(res.outcomes, table, mode)
        fits.append(pr.fit_ols(ex.split_samples(smp)[0]))
    arrs = {"w": np.array([np.append(f.w, f.b) for f in fits]), "alpha": np.array(0.5)}
    profiles = [table.get(models[e // mbs], e % mbs + 1) for e in range(E)]
    for cap in (2, 3, 4):
        own_l, peers_l, yc, yf = [], [], [], []
        rng = np.random.default_rng(cap)
        for own in range(E):
            multisets = [()]
            for k in range(1, cap):
                multisets += list(itertools.combinations_with_replacement(range(E), k))
            if cap >= 3:  # subsample: keep the fixture small
                pick = rng.choice(len(multisets), size=40, replace=False)
                multisets = [multisets[i] for i in sorted(pick)]
            for peers in multisets:
                colo0 = np.zeros(3)
                for q in peers:
                    colo0 = colo0 + profiles[q].throughputs()
                hist = [colo0]
                remaining = list(peers)
                order = sorted((solo[q], q, j) for j, q in enumerate(peers) if solo[q] < solo[own])
                for _, q, j in order:
                    remaining.remove(q)
                    c = np.zeros(3)
                    for r in remaining:
                        c = c + profiles[r].throughputs()
                    hist.append(c)
                est_s = estimate_from_history(0, STATIC_MODE, hist)
                est_f = estimate_from_history(0, ewma_mode(0.5), hist)
                xs = finalize_features(profiles[own], est_s)
                xf = finalize_features(profiles[own], est_f)
                own_l.append(own)
                peers_l.append(list(peers) + [-1] * (cap - 1 - len(peers)))
                yc.append(pr.predict(fits[0], xs))
                yf.append(pr.predict(fits[1], xf))
        arrs[f"cap{cap}/own"] = np.array(own_l, dtype=np.int32)
        arrs[f"cap{cap}/peers"] = np.array(peers_l, dtype=np.int32).reshape(len(own_l), cap - 1)
        arrs[f"cap{cap}/y_coarse"] = np.array(yc)
        arrs[f"cap{cap}/y_fine"] = np.array(yf)
        print(f"candidates cap{cap}: {len(own_l)}")
    np.savez_compressed(os.path.join(HERE, "candidates_golden.npz"), **arrs)


def c5eval_golden(table, n_scen: int = 24):
    """C5 per-scenario evaluation (coarse = static + OLS, fine =
    EWMA(1/2) + OLS, adaptive = OLS warm start + RLS prequential on the 25%
    tail) by the reference's own functions on the bench's scenario generator
    (`paper_2512_18725_b200.sweep.c5_scenario`, host config code only)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2512_18725_b200.sweep import c5_scenario

    from intfsim.workload import scenario_from_dict

    arrs = {"idx": np.arange(n_scen)}
    reps = np.full((n_scen, 3, 6), np.nan)
    for i in range(n_scen):
        spec = scenario_from_dict(c5_scenario(table, i))
        res = intfsim.run_scenario(spec, table)
        s_st = intfsim.colocation.samples_from_outcomes(res.outcomes, table, STATIC_MODE)
        s_ew = intfsim.colocation.samples_from_outcomes(res.outcomes, table, ewma_mode(0.5))
        try:
            tr_s, te_s = ex.split_samples(s_st)
            tr_f, te_f = ex.split_samples(s_ew)
            coarse, fine = pr.fit_ols(tr_s), pr.fit_ols(tr_f)
        except (ValueError, pr.PredictError):
            continue  # too few samples: the reference raises, the device reports NaN / n = 0
        st = pr.rls_init(fine, lam=0.99, X_train=np.array([s.x for s in tr_f]))
        for k, rep in enumerate([pr.evaluate(coarse, te_s), pr.evaluate(fine, te_f), pr.evaluate(st, te_f, online=True)]):
            reps[i, k] = [rep.mse, rep.rel_p25, rep.rel_p50, rep.rel_p75, rep.rel_p95, rep.n_samples]
    arrs["reports"] = reps
    print(f"c5eval: {n_scen} scenarios, {int(np.isnan(reps[:, 0, 0]).sum())} without a valid split")
    np.savez_compressed(os.path.join(HERE, "c5eval_golden.npz"), **arrs)


def main():
    table = load_profiles("/root/reference/pkg/profiles/default.csv")
    assert table.entries == gen_synthetic_profiles().entries
    if "--candidates" in sys.argv:  # only candidates_golden.npz
        candidates_golden(table)
        return
    if "--c5eval" in sys.argv:  # only c5eval_golden.npz
        c5eval_golden(table)
        return
    t16 = table16()
    rng_golden()
    replay_golden(table, t16)
    predict_golden(table)
    candidates_golden(table)
    c5eval_golden(table)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
