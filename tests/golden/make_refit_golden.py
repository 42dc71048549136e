"""Freeze the reference's windowed refit ("refit each window", BASELINE
configs[2]): `fit_ols_xy` (`predict.py:53-66`) on consecutive windows of the
EWMA(1/2) samples of the bundled trace, plus a rank-deficient window (ridge
fallback).  -> tests/golden/refit_golden.npz

    python tests/golden/make_refit_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from intfsim.predict import fit_ols_xy  # noqa: E402


def main():
    P = np.load(os.path.join(HERE, "predict_golden.npz"))
    X = np.concatenate([P["ewma/mode2/X"], P["ridge/X"]])
    y = np.concatenate([P["ewma/mode2/y"], P["ridge/y"]])
    arrs = {"X": X, "y": y}
    for W in (8, 24, 64, 100, 256, 333):
        fits = []
        for i in range(0, len(y), W):
            m = fit_ols_xy(X[i:i + W], y[i:i + W])
            fits.append(np.append(m.w, m.b))
        arrs[f"w{W}"] = np.array(fits)
    # a window that is exactly the rank-deficient block (ridge path)
    n0 = len(P["ewma/mode2/y"])
    arrs["ridge_start"] = np.array(n0)
    np.savez_compressed(os.path.join(HERE, "refit_golden.npz"), **arrs)
    print({k: v.shape for k, v in arrs.items()})


if __name__ == "__main__":
    main()
