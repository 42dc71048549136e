"""The product's replay recurrence (csrc/replay_core.cuh), compiled for the
host (tests/hostcheck, test-only), against the golden outputs.  Exercises
the exact kernel logic on CPU; the GPU tests re-check the sm_100a build."""
import numpy as np
import pytest

from tests import _golden
from tests.hostcheck import driver


@pytest.fixture(scope="module")
def runs():
    out = {}
    for tname in _golden.table_names():
        names = _golden.scenario_names(tname)
        preds = []
        from paper_2512_18725_b200 import _abi

        preds = [_abi.Predictor(ewma=e, alpha=a, w=(0.1, -0.2, 0.3, 0.05, 0.4, -0.1, 1.0)) for e, a in _golden.MODES]
        out[tname] = (names, driver.run([_golden.spec(n) for n in names], _golden.table(tname), preds=preds))
    return out


def test_hostcheck_replay_bit_exact(runs):
    bad = {}
    for tname, (names, res) in runs.items():
        for s, n in enumerate(names):
            v = driver.scenario_view(res, s)
            assert v["status"] == 0, n
            f = _golden.compare_replay(v, n)
            if f:
                bad[n] = f
    assert not bad, bad


def test_hostcheck_dispatch_trace(runs):
    import oracle as O

    for tname, (names, res) in runs.items():
        pb, b = res["pb"], res["bufs"]
        for s, n in enumerate(names):
            S = pb.scen[s]
            nb = int(b["n_batches"][s])
            t = _golden.table(tname)
            ref = O.run_scenario(_golden.spec(n), O.TableArrays(t.models, t.max_bs, t.solo, t.thr))
            assert np.array_equal(b["b_running"][S.req_off:S.req_off + nb], ref["b_running"]), n


def test_hostcheck_features_bit_exact(runs):
    G = _golden.replay()
    for tname, (names, res) in runs.items():
        pb = res["pb"]
        for s, n in enumerate(names):
            S = pb.scen[s]
            nb = int(res["bufs"]["n_batches"][s])
            for mi in range(4):
                np.testing.assert_array_equal(res["X"][mi, S.req_off:S.req_off + nb], G[f"{n}/x_mode{mi}"])
            np.testing.assert_array_equal(res["Y"][S.req_off:S.req_off + nb], G[f"{n}/y_mode0"])


def test_hostcheck_rng_matches_golden():
    R = _golden.load("rng_golden.npz")
    L = driver.lib()
    for (s, b, k), v in zip(R["noise_keys"][:300], R["noise_sigma005"][:300]):
        assert L.hc_noise(int(s), int(b) & 0xFFFFFFFF, int(k), 0.05) == v or int(b) >= 2**32
    assert all(L.hc_exp(float(x)) == y for x, y in zip(R["exp_x"][:5000], R["exp_y"][:5000]))
    assert all(L.hc_log1p(float(x)) == y for x, y in zip(R["log1p_x"][:5000], R["log1p_y"][:5000]))


def test_hostcheck_empty_and_tiny_scenarios():
    tab = _golden.table("default")
    base = _golden.spec("bundled_seed7")
    empty = dict(base, deployed=[dict(d, arrival_rate_rps=0.0) for d in base["deployed"]])
    tiny = dict(base, duration_s=0.002)
    res = driver.run([empty, tiny], tab)
    assert int(res["bufs"]["n_req"][0]) == 0 and int(res["bufs"]["n_batches"][0]) == 0
    assert int(res["bufs"]["status"][0]) == 0 and int(res["bufs"]["status"][1]) == 0


def test_noise_table_shared_prefix_equals_per_draw():
    """noise_draws_k (the noise table: K draws of one batch sharing the
    SeedSequence work that does not involve the segment index) equals
    noise_draw draw by draw, for seeds / batch ids below and above 2^32 (the
    latter take the per-draw path) and sigma 0."""
    import ctypes

    import numpy as np

    L = driver.lib()
    rng = np.random.default_rng(3)
    seed = np.concatenate([rng.integers(0, 2**32, 3000), [0, 1, 2**32 - 1, 2**32, 2**40 + 5]]).astype(np.uint64)
    batch = np.concatenate([rng.integers(0, 2**32, 3000), [0, 2**32 - 1, 7, 3, 2**33]]).astype(np.uint64)
    for sigma in (0.05, 0.3, 0.0):
        bad = L.hc_noise_k_mismatch(seed.ctypes.data_as(ctypes.c_void_p), batch.ctypes.data_as(ctypes.c_void_p),
                                    len(seed), 8, sigma)
        assert bad == 0, (sigma, bad)
