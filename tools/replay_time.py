"""Experiment (tools/): C5-shape whole-scenario replay time per step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_18725_b200 import engine
from paper_2512_18725_b200.profiles import gen_synthetic_profiles
from paper_2512_18725_b200.sweep import c5_scenarios

table = gen_synthetic_profiles()
NK = [int(a) for a in os.environ.get("NOISE_K", "4").split(",")]
for n, nk in [(int(a), k) for a in (sys.argv[1:] or ["10000"]) for k in NK]:
    specs = c5_scenarios(table, n, start=0)
    specs.sort(key=lambda d: -sum(m["arrival_rate_rps"] for m in d["deployed"]) * d["duration_s"])
    pipe = engine.ReplayPipeline(specs, table.arrays(), scale=1.5, noise_k=nk)
    for _ in range(2):
        pipe.run()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    for _ in range(5):
        pipe.run()
    e[1].record()
    torch.cuda.synchronize()
    ms = e[0].elapsed_time(e[1]) / 5
    print(f"n={n} noise_k={nk} {ms:.3f} ms/step {n / ms * 1e3:.0f} replays/s status_nonzero={int((pipe.status() != 0).sum())}")
