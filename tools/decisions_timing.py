"""Real-decision scoring on a replayed 10^4-scenario sweep: dispatch sets vs
scoring (enumeration layout / decision-major features)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_18725_b200 import engine  # noqa: E402
from paper_2512_18725_b200.profiles import gen_synthetic_profiles  # noqa: E402
from paper_2512_18725_b200.sweep import c2_decision_coefs, c5_scenarios, lpt_order  # noqa: E402

table = gen_synthetic_profiles()
ta = table.arrays()
pipe = engine.ReplayPipeline(lpt_order(c5_scenarios(table, 10000)), ta, scale=1.5)
pipe.run()
sc = engine.CandidateScorer(ta, cap=4, alpha=0.5)
coefs = torch.tensor(c2_decision_coefs(32)[-1], device="cuda").contiguous()


def timed(f, reps=10):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


sc.prepare()
rank, own = sc.dispatch_decisions(pipe)
print("decisions", int((rank >= 0).sum()))
print("dispatch_sets", round(timed(lambda: sc.dispatch_decisions(pipe)), 3), "ms")
best, chosen = sc.score_decisions(coefs, rank, own)
print("score (enumeration layout)", round(timed(lambda: sc.score_decisions(coefs, rank, own, best, chosen)), 3), "ms")
sc.prepare_decisions()
print("score (decision-major)", round(timed(lambda: sc.score_decisions(coefs, rank, own, best, chosen)), 3), "ms")
