"""One drift_experiments call over seeds 0..19 (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_18725_b200 as p  # noqa: E402
from paper_2512_18725_b200 import experiments as ex  # noqa: E402

table = p.gen_synthetic_profiles()
ex.drift_experiments([ex.default_drift_base(table, s) for s in range(20)], table)
torch.cuda.synchronize()
