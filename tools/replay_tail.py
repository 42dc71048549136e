"""Experiment (tools/): is the C5 replay step tail-bound?  Times the longest
scenarios alone and the sweep at growing sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_18725_b200 import engine
from paper_2512_18725_b200.profiles import gen_synthetic_profiles
from paper_2512_18725_b200.sweep import c5_scenarios

table = gen_synthetic_profiles()
ta = table.arrays()


def t_run(specs, reps=3):
    pipe = engine.ReplayPipeline(specs, ta, scale=1.5)
    pipe.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pipe.run()
    e1.record()
    torch.cuda.synchronize()
    nb = pipe.t["n_batches"][: pipe.pb.n_scen].cpu().numpy()
    return e0.elapsed_time(e1) / reps, nb


specs = c5_scenarios(table, 10000)
ms, nb = t_run(specs)
order = np.argsort(-nb)
print(f"all 10000: {ms:.3f} ms; batches max {nb.max()} mean {nb.mean():.0f}")
for k in (1, 4, 32, 148, 592, 2368):
    sub = [specs[i] for i in order[:k]]
    ms, _ = t_run(sub)
    print(f"longest {k}: {ms:.3f} ms (min batches in set {nb[order[k - 1]]})")
for n in (20000, 80000):
    ms, _ = t_run(c5_scenarios(table, n))
    print(f"n={n}: {ms:.3f} ms, {n / ms * 1e3:.0f} replays/s")
