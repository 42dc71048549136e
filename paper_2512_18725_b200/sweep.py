"""Synthetic workloads of the benchmark configs, as scenario
dicts ready for the batched device pipeline.

C5: scenario i draws from default_rng([2512, i]): 2-4 models of the bundled
table, total load rho ~ U(0.3, 0.9) split evenly, SLO = U(5, 50) x solo(bs=1),
1 s, window U(0, 10) ms, cap in {1, 2, 3}, sigma 0.05, oracle seed i.
C4: 16 models (6 default archetypes + 10 from default_rng(123)), bs <= 64,
cap 4, heterogeneous per-model load.
"""
from __future__ import annotations

import numpy as np

from .profiles import DEFAULT_ARCHETYPES, Archetype, gen_synthetic_profiles

# C1: the reference's bundled trace `pkg/scenarios/mixed_three_model.json` (3 models, cap 2, seed 7)
BUNDLED_SEED7 = {
    "name": "mixed_three_model", "duration_s": 5.0, "batching_window_ms": 4.0, "max_batch_size": 8,
    "concurrency_cap": 2, "seed": 7, "colocation_mode": "static", "ewma_alpha": 1.0,
    "oracle": {"beta_l2": 1.0, "beta_dram": 1.5, "beta_sm": 0.5, "noise_sigma": 0.05, "seed": 0},
    "deployed": [{"model_id": "resnet50", "arrival_rate_rps": 588.2352941176472, "slo_ms": 10.0},
                 {"model_id": "roberta_b", "arrival_rate_rps": 52.70834726810264, "slo_ms": 30.0},
                 {"model_id": "vit_b16", "arrival_rate_rps": 116.95906432748538, "slo_ms": 22.5}],
}


def c5_scenario(table, i: int) -> dict:
    rng = np.random.default_rng([2512, i])
    models = table.models()
    k = int(rng.integers(2, 5))
    chosen = [models[j] for j in rng.choice(len(models), size=k, replace=False)]
    rho = float(rng.uniform(0.3, 0.9))
    dep = []
    for m in chosen:
        bs = table.max_batch_size
        cap_rps = bs / (table.get(m, bs).solo_duration_ms / 1000.0)
        dep.append({"model_id": m, "arrival_rate_rps": rho / k * cap_rps,
                    "slo_ms": float(rng.uniform(5.0, 50.0)) * table.get(m, 1).solo_duration_ms})
    return {
        "name": f"c5_{i}", "duration_s": 1.0, "batching_window_ms": float(rng.uniform(0.0, 10.0)),
        "max_batch_size": 8, "concurrency_cap": int(rng.integers(1, 4)), "seed": i,
        "colocation_mode": "static", "ewma_alpha": 1.0,
        "oracle": {"beta_l2": 1.0, "beta_dram": 1.5, "beta_sm": 0.5, "noise_sigma": 0.05, "seed": i},
        "deployed": dep,
    }


def c5_scenarios(table, n: int, start: int = 0) -> list:
    return [c5_scenario(table, i) for i in range(start, start + n)]


def expected_requests(spec: dict) -> float:
    """lambda*T of a scenario dict: its expected request count (shard weight)."""
    return sum(d["arrival_rate_rps"] for d in spec["deployed"]) * spec["duration_s"]


def lpt_order(specs: list) -> list:
    """Longest-processing-time first by expected requests (stable): the
    heaviest scenarios get the first replay warps."""
    return sorted(specs, key=lambda d: -expected_requests(d))


def table16():
    rng = np.random.default_rng(123)
    arch = list(DEFAULT_ARCHETYPES)
    for i in range(10):
        base = float(rng.uniform(0.8, 8.0))
        eff = float(rng.uniform(0.2, 0.95))
        mix = tuple(float(v) for v in rng.uniform(0.2, 0.6, size=3))
        arch.append(Archetype(f"synth_{i:02d}", base, eff, mix))
    return gen_synthetic_profiles(arch, seed=0, max_batch_size=64), arch


def c4_scenario(table16_, arch, n_requests: float = 1e6, rho: float = 0.5, seed: int = 1) -> dict:
    """C4: one multi-tenant trace of ~n_requests over 16 models, bs <= 64, cap 4,
    window 10-20 ms, sigma 0.05, oracle seed 1; heterogeneous per-model load
    (total utilisation rho at bs 64) so that light models reach large
    batches and the GPU has many busy periods."""
    rng = np.random.default_rng([4, seed])
    share = rng.uniform(0.5, 1.5, size=len(arch))
    share = share / share.sum()
    dep = []
    for a, f in zip(arch, share):
        solo64 = table16_.get(a.model_id, 64).solo_duration_ms
        rate = rho * f * 64 / (solo64 / 1000.0)
        dep.append({"model_id": a.model_id, "arrival_rate_rps": float(rate),
                    "slo_ms": float(20.0 * table16_.get(a.model_id, 1).solo_duration_ms)})
    total = sum(d["arrival_rate_rps"] for d in dep)
    return {
        "name": "c4", "duration_s": float(n_requests / total), "batching_window_ms": float(rng.uniform(10.0, 20.0)),
        "max_batch_size": 64, "concurrency_cap": 4, "seed": seed, "colocation_mode": "static", "ewma_alpha": 1.0,
        "oracle": {"beta_l2": 1.0, "beta_dram": 1.5, "beta_sm": 0.5, "noise_sigma": 0.05, "seed": 1},
        "deployed": dep,
    }


def c2_decision_coefs(n_dec: int, alpha: float = 0.5) -> np.ndarray:
    """C2 decisions: [n_dec][2][7] coarse (static) / fine (EWMA alpha) OLS
    refits (`predict.py:53-72`) on growing windows of the bundled trace's
    samples (`mixed_three_model.json`, seed 7) -- the coefficients a
    scheduler refitting as samples arrive would hold at n_dec decisions."""
    from . import engine
    from .colocation import STATIC_MODE, ewma_mode, features_for_modes
    from .simcore import run_scenario
    from .workload import scenario_from_dict

    table = gen_synthetic_profiles()
    res = run_scenario(scenario_from_dict(BUNDLED_SEED7), table)
    X, y, _ = features_for_modes(res.outcomes, table, [STATIC_MODE, ewma_mode(alpha)])
    n = len(y)
    W = np.zeros((n_dec, 2, 7))
    for d in range(n_dec):
        hi = max(64, int(n * (d + 1) / n_dec))
        for k in range(2):
            params, _, _, _ = engine.ols_solve(engine.ols_stats(X[k, :hi], y[:hi]))
            W[d, k] = params
    return W
