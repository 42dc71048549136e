"""Single-trace latency: whole-scenario warp replay vs busy-period-sharded
replay (speculative jobs) for the bundled trace (C1) and a drift scenario (C3)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_18725_b200 as p  # noqa: E402
from paper_2512_18725_b200 import _abi, engine  # noqa: E402
from paper_2512_18725_b200 import experiments as ex  # noqa: E402
from paper_2512_18725_b200.sweep import BUNDLED_SEED7  # noqa: E402

table = p.gen_synthetic_profiles()
ta = table.arrays()
cases = {"bundled": [BUNDLED_SEED7], "drift0 (4 scen)": ex.drift_specs(ex.default_drift_base(table, 0)),
         "drift 0..19 (80 scen)": [d for s in range(20) for d in ex.drift_specs(ex.default_drift_base(table, s))]}
pred = [_abi.Predictor(ewma=1, alpha=0.5, w=(0.0,) * 7)]


def timed(f, reps=10):
    f()
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, specs in cases.items():
    pipe = engine.ReplayPipeline(specs, ta, preds=pred, scale=1.5)
    print(name, "batches", None, "whole-scenario warp:", round(timed(pipe.run), 3), "ms")
    for min_len in (8, 16, 32, 96):
        for passes in (3, 4):
            pp = engine.ReplayPipeline(specs, ta, preds=pred, scale=1.5)
            def f():
                fin = engine.replay_segmented(pp, min_len=min_len, passes=passes, stats=False)
                fin()
            ms = timed(f)
            st = engine.replay_segmented(pp, min_len=min_len, passes=passes)
            print(f"  segmented min_len {min_len:3d} passes {passes}: {ms:.3f} ms  jobs {st.get('jobs_initial')}->{st.get('jobs_final')} iters {st.get('iterations')}")
