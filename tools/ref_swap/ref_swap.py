"""pytest plugin: run the reference's own test suite (`pkg/tests`) against
this package through INTEGRATION.md's module swap, on a B200.

    tools/ref_swap/run.sh          # stage (build container) + run (GPU box)

The swap aliases `intfsim` and its submodules to `paper_2512_18725_b200`
before any test module imports them.  Nothing of the reference's own code is
imported: only its tests (staged, git-ignored, under baseline/_ref/pkg/tests).
"""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

pkg = importlib.import_module("paper_2512_18725_b200")
sys.modules["intfsim"] = pkg
for sub in ("batcher", "colocation", "experiments", "metrics", "oracle", "predict", "profiles", "simcore", "workload"):
    sys.modules[f"intfsim.{sub}"] = importlib.import_module(f"paper_2512_18725_b200.{sub}")
