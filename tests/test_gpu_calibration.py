"""Device calibration drivers (`experiments.py:255-329`) against the
reference's outputs: full_overlap_ratios as one batched replay of n_pairs
scenarios (noise key offset batch_id_base = 2k), bit-exact; calibration_p95;
stress-scenario p99 latency through run_scenario."""
import json

import numpy as np
import pytest

from tests import _golden

pytestmark = pytest.mark.gpu
CASES = ["default", "mixed_bs4", "light_sigma0", "heavy_sigma0", "convnext_vgg"]


def _table():
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles

    return gen_synthetic_profiles()


@pytest.mark.parametrize("name", CASES)
def test_full_overlap_ratios_bit_exact(name):
    from paper_2512_18725_b200 import experiments
    from paper_2512_18725_b200.interference import InterferenceOracle

    g = _golden.load("calib_golden.npz")
    a = json.loads(str(g[name + "/args"]))
    orc = InterferenceOracle(**a["oracle"])
    kw = dict(model_a=a["model_a"], model_b=a["model_b"], batch_size=a["batch_size"], n_pairs=a["n_pairs"],
              oracle=orc)
    r = experiments.full_overlap_ratios(_table(), **kw)
    np.testing.assert_array_equal(np.array(r), g[name + "/ratios"])
    assert experiments.calibration_p95(_table(), **kw) == float(g[name + "/p95"])


@pytest.mark.parametrize("cap", [1, 2, 3])
def test_stress_p99_latency(cap):
    import paper_2512_18725_b200 as intfsim
    from paper_2512_18725_b200 import experiments

    t = _table()
    s = experiments.symmetric_stress_scenario(t, ["resnet50", "yolov8n"], 1.1, 3, cap)
    p99 = experiments.p99_latency(intfsim.run_scenario(s, t).records)
    assert p99 == float(_golden.load("calib_golden.npz")[f"stress{cap}/p99"])
