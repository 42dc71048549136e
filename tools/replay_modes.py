"""Experiment (tools/): C5-shape sweep replayed whole-scenario-per-warp
(pipe.run) vs busy-period sharded (engine.replay_segmented), per step time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_18725_b200 import engine
from paper_2512_18725_b200.profiles import gen_synthetic_profiles
from paper_2512_18725_b200.sweep import c5_scenarios

table = gen_synthetic_profiles()
ta = table.arrays()
for n in (4096, 10000):
    specs = c5_scenarios(table, n, start=0)
    specs.sort(key=lambda d: -sum(m["arrival_rate_rps"] for m in d["deployed"]) * d["duration_s"])
    pipe = engine.ReplayPipeline(specs, ta, scale=1.5)
    pipe.run()
    torch.cuda.synchronize()
    ref = {k: pipe.t[k].clone() for k in ("b_start", "b_completion", "r_batch", "out_order")}

    def timed(f, reps=5):
        f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            r = f()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) / reps * 1e3, r

    ms, wall, _ = timed(pipe.run)
    print(f"n={n} whole-scenario: {ms:.3f} ms/step ({n / ms * 1e3:.0f} replays/s) wall {wall:.3f}")
    for slow, ml in ((2.0, 16), (2.0, 4), (1.5, 8), (3.0, 16), (2.0, 64)):
        ms, wall, st = timed(lambda: engine.replay_segmented(pipe, slow=slow, min_len=ml))
        same = all(torch.equal(pipe.t[k], ref[k]) for k in ref)
        print(f"n={n} segmented slow={slow} min_len={ml}: {ms:.3f} ms/step ({n / ms * 1e3:.0f} replays/s) "
              f"wall {wall:.3f} same={same} {st}")
