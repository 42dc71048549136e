"""Freeze the reference's fit_ols_xy (`predict.py:53-66`) on ill-conditioned
and rank-deficient designs -- where matrix_rank(Z) and lstsq, not the
normal equations, decide the result: every row identical (the reference's own
`test_ols_ridge_fallback_on_collinear_design`), a constant feature, exactly
proportional features, duplicated rows in a short design, a nearly collinear
full-rank design, a constant feature over 2*10^5 rows (multi-block QR), and a
well-conditioned control (designs regenerated from a seed by
ols_rank_designs.py, so only the results are stored).
-> tests/golden/ols_rank_golden.npz

    python tests/golden/make_ols_rank_golden.py
"""
from __future__ import annotations

import logging
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from intfsim.predict import fit_ols_xy  # noqa: E402

sys.path.insert(0, HERE)
from ols_rank_designs import designs  # noqa: E402


def main():
    logging.disable(logging.WARNING)
    arrs = {}
    for name, (X, y) in designs().items():
        Z = np.column_stack([X, np.ones(len(X))])
        m = fit_ols_xy(X, y)
        arrs[f"{name}/params"] = np.append(m.w, m.b)
        arrs[f"{name}/ridge"] = np.array(np.linalg.matrix_rank(Z) < 7)
        print(name, X.shape, "ridge" if arrs[f"{name}/ridge"] else "lstsq", "cond(Z) %.2e" % np.linalg.cond(Z))
    np.savez_compressed(os.path.join(HERE, "ols_rank_golden.npz"), **arrs)


if __name__ == "__main__":
    main()
