"""Freeze the reference's calibration-driver outputs (`experiments.py:255-329`)
into tests/golden/calib_golden.npz (unmodified reference, this container).

    python tests/golden/make_calib_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import intfsim  # noqa: E402
from intfsim import experiments as ex  # noqa: E402
from intfsim.oracle import InterferenceOracle  # noqa: E402
from intfsim.workload import scenario_to_dict  # noqa: E402

CASES = {
    # name: (model_a, model_b, batch_size, n_pairs, oracle kwargs)
    "default": ("roberta_b", "roberta_b", 8, 200, {}),
    "mixed_bs4": ("resnet50", "yolov8n", 4, 60, {"seed": 3, "noise_sigma": 0.1}),
    "light_sigma0": ("yolov8n", "resnet50", 1, 20, {"noise_sigma": 0.0}),
    "convnext_vgg": ("convnext_b", "vgg19", 2, 30, {"seed": 11}),
    "heavy_sigma0": ("vit_b16", "roberta_b", 8, 20, {"noise_sigma": 0.0, "seed": 5}),
}


def main():
    table = intfsim.load_profiles("/root/reference/pkg/profiles/default.csv")
    arrs = {}
    for name, (a, b, bs, n, okw) in CASES.items():
        orc = InterferenceOracle(**okw)
        r = ex.full_overlap_ratios(table, model_a=a, model_b=b, batch_size=bs, n_pairs=n, oracle=orc)
        arrs[name + "/ratios"] = np.array(r)
        arrs[name + "/args"] = np.array(json.dumps({"model_a": a, "model_b": b, "batch_size": bs, "n_pairs": n,
                                                    "oracle": okw}))
        arrs[name + "/p95"] = np.array(ex.calibration_p95(table, model_a=a, model_b=b, batch_size=bs, n_pairs=n,
                                                          oracle=orc))
    for cap in (1, 2, 3):
        s = ex.symmetric_stress_scenario(table, ["resnet50", "yolov8n"], 1.1, 3, cap)
        arrs[f"stress{cap}/spec"] = np.array(json.dumps(scenario_to_dict(s)))
        arrs[f"stress{cap}/p99"] = np.array(ex.p99_latency(intfsim.run_scenario(s, table).records))
    np.savez_compressed(os.path.join(HERE, "calib_golden.npz"), **arrs)
    print(sorted(arrs))


if __name__ == "__main__":
    main()
