"""bench.py end to end on a B200 (a short run without the CPU baselines): the
driver's contract -- one JSON line with the headline metric, the roofline,
the end-to-end call, clocks and launches -- and every secondary leg (C5 sweep,
C4 long trace, C1 bundled trace, C3 drift, refit rates) present and sane."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu"], cwd=ROOT,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert 0.5 < d["roofline"]["frac"] < 1.2 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["valid"]
    assert d["replay"]["status_nonzero"] == 0 and d["replay"]["eval_invalid"] == 0 and d["replay"]["value"] > 0
    assert d["long_trace"]["status"] == 0 and d["long_trace"]["pipelined"]["complete"]
    for leg in ("bundled_trace", "drift", "refit", "best_step"):
        assert leg in d and d[leg]["value" if leg != "refit" else "rls"], leg
