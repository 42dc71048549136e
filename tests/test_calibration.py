"""Calibration / stress drivers (`experiments.py:255-329`): the
oracle's restatement of full_overlap_ratios against the reference's outputs
(tests/golden/calib_golden.npz, made by tests/golden/make_calib_golden.py),
and the host-side stress-scenario config.  GPU parity of the device path is
in tests/test_gpu_calibration.py."""
import json

import numpy as np
import pytest

import oracle as O
from tests import _golden

CASES = ["default", "mixed_bs4", "light_sigma0", "heavy_sigma0", "convnext_vgg"]


def _gold():
    return _golden.load("calib_golden.npz")


@pytest.mark.parametrize("name", CASES)
def test_oracle_full_overlap_ratios_bit_exact(name):
    g = _gold()
    a = json.loads(str(g[name + "/args"]))
    o = a["oracle"]
    tab = _golden.table("default")
    otab = O.TableArrays(tab.models, tab.max_bs, tab.solo, tab.thr)
    r = O.full_overlap_ratios(otab, a["model_a"], a["model_b"], a["batch_size"], a["n_pairs"],
                              seed=o.get("seed", 0), sigma=o.get("noise_sigma", 0.05))
    np.testing.assert_array_equal(np.array(r), g[name + "/ratios"])
    assert O.percentile(r, 95) == float(g[name + "/p95"])


def test_criterion7_calibration_target():
    """Acceptance criterion 7: p95 of full-overlap roberta_b pairs in [1.4, 1.6]."""
    assert 1.4 <= float(_gold()["default/p95"]) <= 1.6


@pytest.mark.parametrize("cap", [1, 2, 3])
def test_symmetric_stress_scenario_matches_reference(cap):
    from paper_2512_18725_b200.experiments import symmetric_stress_scenario
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles
    from paper_2512_18725_b200.workload import scenario_to_dict

    s = symmetric_stress_scenario(gen_synthetic_profiles(), ["resnet50", "yolov8n"], 1.1, 3, cap)
    assert scenario_to_dict(s) == json.loads(str(_gold()[f"stress{cap}/spec"]))
