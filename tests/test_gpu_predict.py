"""GPU parity of the refit path: OLS statistics + solve, prequential SGD /
RLS streams, evaluation reports, and the experiment drivers, against the
reference's golden outputs.  Tolerance 1e-5 relative (north star); SGD is
additionally checked bit-exact (same rounding sequence as numpy)."""
import numpy as np
import pytest

from tests import _golden

pytestmark = pytest.mark.gpu
RTOL = 1e-5


def _samples(X, y):
    import paper_2512_18725_b200 as p

    return [p.Sample(x=X[i], y=float(y[i]), batch_id=i) for i in range(len(y))]


def test_fit_ols_matches_lstsq():
    import paper_2512_18725_b200 as p

    P = _golden.load("predict_golden.npz")
    for mi in range(4):
        X, y, cut = P[f"ewma/mode{mi}/X"], P[f"ewma/mode{mi}/y"], int(P[f"ewma/mode{mi}/ncut"])
        m = p.fit_ols(_samples(X[:cut], y[:cut]))
        np.testing.assert_allclose(m.w7(), np.append(P[f"ewma/mode{mi}/w"], P[f"ewma/mode{mi}/b"]), rtol=RTOL,
                                   atol=1e-9)
        rep = p.evaluate(m, _samples(X[cut:], y[cut:]))
        np.testing.assert_allclose([rep.mse, rep.rel_p25, rep.rel_p50, rep.rel_p75, rep.rel_p95, rep.n_samples],
                                   P[f"ewma/mode{mi}/report"], rtol=RTOL)


def test_ridge_fallback_when_rank_deficient():
    import paper_2512_18725_b200 as p

    P = _golden.load("predict_golden.npz")
    m = p.fit_ols_xy(P["ridge/X"], P["ridge/y"])
    np.testing.assert_allclose(m.w7(), P["ridge/w"], rtol=RTOL, atol=1e-7)


def test_exact_recovery_and_rls_equals_ols():
    # `test_predict.py:45-50` and criterion 1 (`test_acceptance.py:45-65`)
    import paper_2512_18725_b200 as p

    rng = np.random.default_rng(0)
    w_true = np.array([0.5, -0.2, 0.8, 0.1, 0.3, -0.4])
    X = rng.uniform(0, 2, size=(200, 6))
    y = X @ w_true + 0.2
    m = p.fit_ols(_samples(X, y))
    np.testing.assert_allclose(m.w, w_true, atol=1e-8)
    y2 = y + 0.2 * rng.standard_normal(200)
    s = _samples(X, y2)
    st = p.rls_init(p.fit_ols(s[:80]), lam=1.0, X_train=X[:80])
    p.evaluate(st, s[80:], online=True)
    full = p.fit_ols(s)
    np.testing.assert_allclose(st.model.w7(), full.w7(), atol=1e-8)


def test_prequential_streams_match_golden():
    import paper_2512_18725_b200 as p

    P = _golden.load("predict_golden.npz")
    for seed in (0, 1):
        pre = f"drift{seed}/"
        m0 = p.LinearModel(w=P[pre + "w0"].copy(), b=float(P[pre + "b0"]))
        Xtr = P[pre + "Xtrain"]
        rls0 = p.rls_init(m0, lam=0.99, X_train=Xtr)
        np.testing.assert_allclose(rls0.P, P[pre + "P0"], rtol=1e-6, atol=1e-6 * np.abs(P[pre + "P0"]).max())
        for ts in ("TestSet1", "TestSet2", "TestSet3"):
            X, y = P[pre + ts + "/X"], P[pre + ts + "/y"]
            sgd = p.SgdState(m0.copy(), eta=0.01)
            rls = rls0.copy()
            rs = p.evaluate_many([sgd, rls], [_samples(X, y)] * 2, online=True)
            np.testing.assert_array_equal(sgd.model.w7(), P[pre + ts + "/sgd_w"])  # bit-exact
            np.testing.assert_allclose(rls.model.w7(), P[pre + ts + "/rls_w"], rtol=RTOL, atol=1e-8)
            ref = p.evaluate(p.SgdState(m0.copy(), eta=0.01), _samples(X, y), online=True)
            assert rs[0] == ref


def test_drift_experiment_matches_reference():
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import experiments as ex

    P = _golden.load("predict_golden.npz")
    table = p.gen_synthetic_profiles()
    for seed in (0, 1):
        cells = ex.drift_experiment(ex.default_drift_base(table, seed), table)
        keys = [f"{c.dataset}/{c.method}" for c in cells]
        assert keys == [str(k) for k in P[f"drift{seed}/cell_keys"]]
        np.testing.assert_allclose([[c.mse, c.n_samples] for c in cells], P[f"drift{seed}/cells"], rtol=RTOL)


def test_ewma_experiment_matches_reference():
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import experiments as ex

    P = _golden.load("predict_golden.npz")
    table = p.gen_synthetic_profiles()
    rows = ex.ewma_experiment(ex.high_churn_suite(table, 0), table)
    for mi, row in enumerate(rows):
        r = row.report
        np.testing.assert_allclose([r.mse, r.rel_p25, r.rel_p50, r.rel_p75, r.rel_p95, r.n_samples],
                                   P[f"ewma/mode{mi}/report"], rtol=RTOL)


@pytest.mark.parametrize("name", ["identical", "constant", "proportional", "duplicates", "near_collinear",
                                  "constant_big", "control"])
def test_fit_ols_ill_conditioned_matches_reference(name):
    """fit_ols_xy where matrix_rank(Z) and lstsq decide (the reference's
    collinear-design test and friends, tests/golden/ols_rank_golden.npz):
    the device QR of the rows gives the reference's rank (ridge or not) and,
    for the nearly collinear full-rank design, lstsq's accuracy."""
    import logging

    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import engine
    from tests.golden.ols_rank_designs import designs

    from paper_2512_18725_b200.predict import predict

    G = _golden.load("ols_rank_golden.npz")
    X, y = designs()[name]
    params, ridge, nonfinite = engine.ols_fit(X, y)
    ref = G[f"{name}/params"]
    assert ridge == bool(G[f"{name}/ridge"]) and not nonfinite
    if ridge:
        # solve(Z^T Z + 1e-8 I, Z^T y) fixes the component along Z's null
        # direction only through the rounding of Z^T Z and Z^T y (the
        # reference's BLAS order): parity is the ridge decision and the fit
        Z = np.column_stack([X, np.ones(len(y))])
        np.testing.assert_allclose(Z @ params, Z @ ref, rtol=RTOL, atol=1e-7)
    else:
        np.testing.assert_allclose(params, ref, rtol=RTOL, atol=1e-7)
    logging.disable(logging.WARNING)
    try:
        m = p.fit_ols_xy(X, y)
    finally:
        logging.disable(logging.NOTSET)
    np.testing.assert_array_equal(m.w7(), params)
    if name == "identical":  # the reference's test_ols_ridge_fallback_on_collinear_design
        assert abs(predict(m, X[0]) - 1.5) <= 1e-3


@pytest.mark.parametrize("window", [8, 24, 64, 100, 256, 333])
def test_windowed_refit_matches_reference(window):
    """Refit each window (BASELINE configs[2]): one statistics + one solve
    launch for every window vs the reference's fit_ols_xy per window
    (tests/golden/refit_golden.npz), incl. a rank-deficient (ridge) window and
    a 1-row tail window."""
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200.predict import fit_ols_windows

    R = _golden.load("refit_golden.npz")
    fits = fit_ols_windows(R["X"], R["y"], window)
    got = np.array([m.w7() for m in fits])
    ref = R[f"w{window}"]
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=RTOL, atol=1e-7)
    # the first window equals the single-fit path
    m0 = p.fit_ols_xy(R["X"][:window], R["y"][:window])
    np.testing.assert_allclose(got[0], m0.w7(), rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("eps", [1e-5, 1e-6, 0.0])
def test_rls_init_p0_near_collinear_matches_numpy_inv(eps):
    """rls_init's P0 = np.linalg.inv(Z^T Z) (`predict.py:126-131`): LU with
    partial pivoting, ridge only on an exactly singular design (eps = 0: two
    identical columns, numpy's LinAlgError -> inv(G + 1e-8 I)).  At cond(G)
    5.8e10 / 4.5e12 the reference's P0 differs from the ridge form by 43% / 98%,
    so a Cholesky-failure ridge would be visible here."""
    import paper_2512_18725_b200 as p

    rng = np.random.default_rng(3)
    X = rng.uniform(0, 1, size=(300, 6))
    X[:, 5] = X[:, 4] + eps * rng.standard_normal(300)
    Z = np.column_stack([X, np.ones(300)])
    G = Z.T @ Z
    try:
        ref = np.linalg.inv(G)
    except np.linalg.LinAlgError:
        ref = np.linalg.inv(G + 1e-8 * np.eye(7))
    st = p.rls_init(p.LinearModel(w=np.zeros(6), b=0.0), X_train=X)
    # the device's Z^T Z sums in another order: P0 moves by ~cond(G) * eps_64 relative
    tol = {1e-5: 1e-3, 1e-6: 3e-2, 0.0: 1e-4}[eps]
    assert np.linalg.norm(st.P - ref) / np.linalg.norm(ref) < tol


def test_batched_drift_equals_per_seed():
    """drift_experiments over several bases (one batched device flow) equals
    drift_experiment per base, bit for bit."""
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import experiments as ex

    table = p.gen_synthetic_profiles()
    bases = [ex.default_drift_base(table, s) for s in (3, 4, 5)]
    together = ex.drift_experiments(bases, table)
    for b, cells in zip(bases, together):
        alone = ex.drift_experiment(b, table)
        assert [(c.dataset, c.method, c.n_samples) for c in cells] == [(c.dataset, c.method, c.n_samples) for c in alone]
        np.testing.assert_array_equal([c.mse for c in cells], [c.mse for c in alone])
