"""The scalar calls of the per-object API (intf_scalar: arguments as kernel
parameters, results through mapped pinned memory) equal their batched twins
bit for bit: noise draws, slowdowns, predictions, EWMA steps, and whole
per-sample SGD / RLS streams against intf_sgd_streams / intf_rls_streams."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_scalar_ops_equal_batched():
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import engine

    rng = np.random.default_rng(4)
    o = p.InterferenceOracle(noise_sigma=0.07, seed=123)
    keys = rng.integers(0, 10 ** 6, size=(200, 2))
    batched = engine.noise_draws(123, 0.07, keys[:, 0], keys[:, 1])
    assert np.array_equal([o.noise_draw(int(b), int(k)) for b, k in keys], batched)
    own, colo, nz = rng.uniform(0, 1, (200, 3)), rng.uniform(0, 2, (200, 3)), rng.uniform(0.8, 1.2, 200)
    batched = engine.slowdowns(own, colo, o.betas(), nz)
    assert np.array_equal([p.oracle_slowdown(own[i], colo[i], o, nz[i]) for i in range(200)], batched)
    m = p.LinearModel(w=rng.normal(size=6), b=0.3)
    X = rng.uniform(0, 1, (200, 6))
    assert np.array_equal([p.predict.predict(m, x) for x in X], engine.predict_rows(X, m.w7()))
    est = p.init_estimate(0, p.ewma_mode(0.5), colo[0])
    hist = [colo[0]]
    for i in range(1, 20):
        p.observe(est, colo[i])
        hist.append(colo[i])
    assert np.array_equal(est.r_hat, p.colocation._fold(np.array(hist), p.ewma_mode(0.5)))


def test_per_sample_sgd_rls_equal_streams():
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import engine

    rng = np.random.default_rng(9)
    X = rng.uniform(0, 1, (150, 6))
    y = X @ np.array([0.3, 0.5, 0.2, 0.8, 1.1, 0.4]) + 1.0 + 0.02 * rng.standard_normal(150)
    samples = [p.Sample(x=X[i], y=float(y[i]), batch_id=i) for i in range(150)]
    m0 = p.fit_ols(samples[:40])
    sgd = p.SgdState(m0.copy(), eta=0.05)
    rls = p.rls_init(m0, lam=0.97, X_train=X[:40])
    P0 = rls.P.copy()
    for s in samples[40:]:
        p.sgd_update(sgd, s)
        p.rls_update(rls, s)
    _, ps, _ = engine.sgd_streams([X[40:]], [y[40:]], m0.w7()[None], [0.05])
    _, pr, Pr, _ = engine.rls_streams([X[40:]], [y[40:]], m0.w7()[None], P0[None], [0.97])
    assert np.array_equal(sgd.model.w7(), ps[0])
    assert np.array_equal(rls.model.w7(), pr[0]) and np.array_equal(rls.P, Pr[0])


def test_scalar_call_latency():
    """One scalar call is one launch + one synchronisation (measured; the
    bound is generous for a shared box)."""
    import paper_2512_18725_b200 as p

    o = p.InterferenceOracle(noise_sigma=0.05, seed=1)
    for _ in range(20):
        p.oracle_slowdown((0.5, 0.4, 0.3), (0.2, 0.3, 0.1), o, o.noise_draw(3, 1))
    t0 = time.perf_counter()
    for i in range(500):
        p.oracle_slowdown((0.5, 0.4, 0.3), (0.2, 0.3, 0.1), o, o.noise_draw(3, i))
    per = (time.perf_counter() - t0) / 1000
    print(f"scalar call: {1e6 * per:.1f} us")
    assert per < 200e-6
