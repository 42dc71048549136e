"""Seeded ill-conditioned / rank-deficient OLS designs shared by
make_ols_rank_golden.py (reference results) and tests/test_gpu_predict.py."""
import numpy as np


def designs():
    rng = np.random.default_rng(20251218)
    out = {}
    out["identical"] = np.tile([0.4, 0.4, 0.4, 0.2, 0.2, 0.2], (20, 1)), np.full(20, 1.5)
    X = rng.random((500, 6))
    X[:, 0] = 0.37
    out["constant"] = X, X @ [0.3, -1.0, 2.0, 0.5, 0.1, -0.7] + 0.9 + 0.01 * rng.standard_normal(500)
    X = rng.random((300, 6))
    X[:, 2] = 2.0 * X[:, 0]
    out["proportional"] = X, X @ [1.0, 0.5, -0.2, 0.0, 0.3, 1.1] + 0.2 + 0.01 * rng.standard_normal(300)
    base = rng.random((6, 6))
    X = base[[0, 1, 2, 3, 0, 4, 5, 3]]
    out["duplicates"] = X, rng.random(8)
    X = rng.random((400, 6))
    X[:, 2] = X[:, 0] + 1e-7 * rng.standard_normal(400)
    out["near_collinear"] = X, X @ [0.5, 0.1, 0.4, -0.3, 0.2, 0.6] + 1.0 + 0.01 * rng.standard_normal(400)
    X = rng.random((200000, 6))
    X[:, 4] = 0.61
    out["constant_big"] = X, X @ [0.2, 0.2, -0.4, 0.8, 0.0, 0.3] - 0.5 + 0.01 * rng.standard_normal(200000)
    X = rng.random((1000, 6))
    out["control"] = X, X @ [1.0, 2.0, 3.0, -1.0, -2.0, 0.5] + 0.25 + 0.01 * rng.standard_normal(1000)
    return out
