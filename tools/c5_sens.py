"""Experiment (tools/): C5 sweep time in the bench's steady state (several
pipelines on their own streams) with parts toggled, to see which stages are
on the throughput path.  env: PIPES (3), EVAL (1), NOISE_K (6), STEPS (20)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_18725_b200 import _abi, engine  # noqa: E402
from paper_2512_18725_b200.profiles import gen_synthetic_profiles  # noqa: E402
from paper_2512_18725_b200.sweep import c5_scenarios, lpt_order  # noqa: E402

P = int(os.environ.get("PIPES", "3"))
ev = os.environ.get("EVAL", "1") == "1"
nk = int(os.environ.get("NOISE_K", "6"))
steps = int(os.environ.get("STEPS", "20"))
feat = os.environ.get("FEAT", "1") == "1"  # (EVAL=0 only)
slo = os.environ.get("SLO", "1") == "1"
table = gen_synthetic_profiles()
preds = [_abi.Predictor(ewma=0, alpha=1.0, w=(0.0,) * 7), _abi.Predictor(ewma=1, alpha=0.5, w=(0.0,) * 7)]
specs = lpt_order(c5_scenarios(table, 10000))
kw = dict(preds=preds, evaluate=(0, 1, 0.99)) if ev else {}
pipes = [engine.ReplayPipeline(specs, table.arrays(), scale=1.5, noise_k=nk, **kw) for _ in range(P)]
streams = [torch.cuda.Stream() for _ in pipes]
for k in range(P):
    with torch.cuda.stream(streams[k]):
        pipes[k].run()
        pipes[k].run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for s in streams:
    s.wait_event(e0)
for k in range(steps):
    with torch.cuda.stream(streams[k % P]):
        pipes[k % P].run(features=feat, slo=slo)
for s in streams:
    torch.cuda.current_stream().wait_stream(s)
e1.record()
torch.cuda.synchronize()
print(f"PIPES={P} EVAL={int(ev)} FEAT={int(feat)} SLO={int(slo)} NOISE_K={nk}: {e0.elapsed_time(e1) / steps:.3f} ms per sweep")
