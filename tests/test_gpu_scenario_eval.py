"""C5 per-scenario predictor evaluation on B200 (intf_scenario_eval): coarse
(static + OLS), fine (EWMA(1/2) + OLS) and adaptive (OLS warm start + RLS
prequential on the 25% tail) EvalReports per scenario, against the
reference's own functions (tests/golden/c5eval_golden.npz) and the oracle's
composition of them on 400 sweep scenarios.  Tolerance 1e-5 relative."""
import numpy as np
import pytest

import oracle as O
from tests import _golden

pytestmark = pytest.mark.gpu
RTOL = 1e-5


def _run(specs, ta):
    from paper_2512_18725_b200 import _abi, engine

    preds = [_abi.Predictor(ewma=0, alpha=1.0, w=(0.0,) * 7), _abi.Predictor(ewma=1, alpha=0.5, w=(0.0,) * 7)]
    pipe = engine.ReplayPipeline(specs, ta, preds=preds, scale=1.5, evaluate=(0, 1, 0.99))
    pipe.run()
    return pipe, pipe.fetch()


def _close(got, ref):
    """Reports agree to 1e-5 relative; a quantile that is ~0 relative to the
    scenario's error scale (exact fits) is compared against that scale."""
    scale = np.maximum(np.abs(ref), 1e-5 * np.nanmax(np.abs(ref[:, 1:5]), axis=1, keepdims=True))
    return np.all(np.abs(got - ref) <= RTOL * scale)


def _singular_tail(rep, spec, otab) -> bool:
    """The adaptive row starts RLS from P0 = inv(Z^T Z) of the EWMA training
    design (`predict.py:126-131`).  When that design is singular (two deployed
    models whose feature vectors span < 7 dimensions), P0 ~ 1e14 is set by the
    rounding of Z^T Z: the reference's own adaptive report moves by ~2% when
    Z^T Z is merely summed in another order (oracle.gram_rows), so it is not
    determined to 1e-5 and is checked for finiteness only."""
    Xf, y, _ = O.samples_from_replay(rep, spec, otab, True, 0.5)
    cut = int(round(0.75 * len(y)))
    Z = np.column_stack([Xf[:cut], np.ones(cut)])
    return np.linalg.cond(Z.T @ Z) > 1e12


def test_scenario_eval_matches_reference_goldens():
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles
    from paper_2512_18725_b200.sweep import c5_scenario

    G = _golden.load("c5eval_golden.npz")
    table = gen_synthetic_profiles()
    specs = [c5_scenario(table, int(i)) for i in G["idx"]]
    pipe, h = _run(specs, table.arrays())
    for s in range(len(specs)):
        v = pipe.scenario(h, s)
        ref = G["reports"][s]
        assert v["status"] == 0
        if np.isnan(ref[0, 0]):
            assert v["eval_status"] & 1 and np.all(v["eval_report"][:, 5] == 0)
            continue
        assert _close(v["eval_report"], ref), (s, v["eval_report"], ref)


def test_scenario_eval_400_sweep_scenarios_vs_oracle():
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles
    from paper_2512_18725_b200.sweep import c5_scenarios, lpt_order

    table = gen_synthetic_profiles()
    ta = table.arrays()
    specs = lpt_order(c5_scenarios(table, 400, start=5000))
    pipe, h = _run(specs, ta)
    otab = O.TableArrays(ta.models, ta.max_bs, ta.solo, ta.thr)
    bad, n_sensitive = [], 0
    for s, spec in enumerate(specs):
        v = pipe.scenario(h, s)
        rep = O.run_scenario(spec, otab)
        ref = O.scenario_eval(rep, spec, otab)
        if ref is None:
            ok = bool(v["eval_status"] & 1)
        elif _close(v["eval_report"], ref):
            ok = not (v["eval_status"] & 1)
        else:  # only where the reference itself is not determined: a singular EWMA training design
            n_sensitive += 1
            ok = not (v["eval_status"] & 1) and bool(v["eval_status"] & 4) and _singular_tail(rep, spec, otab)
            ok = ok and _close(v["eval_report"][:2], ref[:2])  # coarse and fine still agree to 1e-5
            ok = ok and np.all(np.isfinite(v["eval_report"][2])) and v["eval_report"][2, 5] == ref[2, 5]
        if not ok:
            bad.append((s, spec["name"], v["eval_status"], v["eval_report"], ref))
    assert not bad, bad[:3]
    assert n_sensitive <= len(specs) // 50, n_sensitive  # 1 of these 400
