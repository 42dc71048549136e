"""cProfile of experiments.drift_experiments for seeds 0..19 (C3 e2e)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_18725_b200 as p  # noqa: E402
from paper_2512_18725_b200 import experiments as ex  # noqa: E402

table = p.gen_synthetic_profiles()
bases = [ex.default_drift_base(table, s) for s in range(20)]
ex.drift_experiments(bases[:2], table)
torch.cuda.synchronize()
t0 = time.perf_counter()
ex.drift_experiments(bases, table)
torch.cuda.synchronize()
print(f"drift_experiments 20 seeds: {(time.perf_counter() - t0) * 1e3:.1f} ms")
pr = cProfile.Profile()
pr.enable()
ex.drift_experiments(bases, table)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
