"""One C5 sweep (10^4 scenarios, coarse/fine/adaptive evaluation) for
profiling: `ncu --metrics gpu__time_duration.sum python tools/c5_once.py`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_18725_b200 import _abi, engine  # noqa: E402
from paper_2512_18725_b200.profiles import gen_synthetic_profiles  # noqa: E402
from paper_2512_18725_b200.sweep import c2_decision_coefs, c5_scenarios, lpt_order  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
table = gen_synthetic_profiles()
# C5_ONCE_PLAIN=1: zero coefficients (no bundled-trace replay before the sweep: the
# sweep's launches are then the first of each kernel, for ncu -c 1)
W = np.zeros((1, 2, 7)) if os.environ.get("C5_ONCE_PLAIN") else c2_decision_coefs(32)
preds = [_abi.Predictor(ewma=0, alpha=1.0, w=tuple(W[-1, 0])), _abi.Predictor(ewma=1, alpha=0.5, w=tuple(W[-1, 1]))]
pipe = engine.ReplayPipeline(lpt_order(c5_scenarios(table, n)), table.arrays(), preds=preds, scale=1.5,
                             evaluate=(0, 1, 0.99))
pipe.run()
torch.cuda.synchronize()
print("status", int((pipe.status() != 0).sum()), "eval_invalid", int((pipe.eval_status.cpu().numpy()[:n] & 1).sum()))
