"""Experiment (tools/): whole C4 trace time (engine.replay_segmented with
queued passes, as bench.py) vs the speculation parameters (slow, min_len);
best of 5 per setting."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_18725_b200 import engine
from paper_2512_18725_b200.sweep import c4_scenario, table16

t16, arch = table16()
seed = int(os.environ.get("SEED", "1"))
spec = c4_scenario(t16, arch, n_requests=1e6, seed=seed)
ta = t16.arrays()
slows = [float(x) for x in os.environ.get("SLOWS", "1.5,2.0,2.5,3.0").split(",")]
mls = [int(x) for x in os.environ.get("MIN_LENS", "32,64,96,128,192").split(",")]
print(f"seed {seed}")
for slow in slows:
    for ml in mls:
        pipe = engine.ReplayPipeline([spec], ta, scale=1.2)
        st = engine.replay_segmented(pipe, slow=slow, min_len=ml, passes=4)
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = engine.replay_segmented(pipe, slow=slow, min_len=ml, passes=4)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"slow={slow} min_len={ml}: {best:.3f} ms  jobs {st['jobs_initial']} -> {st['jobs_final']}, "
              f"iterations {st['iterations']}", flush=True)
