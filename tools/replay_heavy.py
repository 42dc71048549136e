"""Experiment (tools/): the heaviest C5 scenarios replayed whole (one warp each)
vs busy-period sharded (engine.replay_segmented)."""
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
specs = c5_scenarios(table, 10000)
pipe = engine.ReplayPipeline(specs, ta, scale=1.5)
pipe.run()
nb = pipe.t["n_batches"][: pipe.pb.n_scen].cpu().numpy()
order = np.argsort(-nb)


def timed(f, reps=3):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


for k in (16, 64, 256):
    sub = [specs[i] for i in order[:k]]
    p1 = engine.ReplayPipeline(sub, ta, scale=1.5)
    ms1, _ = timed(p1.run)
    for ml in (16, 64):
        p2 = engine.ReplayPipeline(sub, ta, scale=1.5)
        ms2, st = timed(lambda: engine.replay_segmented(p2, min_len=ml))
        print(f"top {k} (batches >= {nb[order[k - 1]]}): whole {ms1:.3f} ms, segmented(min_len={ml}) {ms2:.3f} ms {st}")
