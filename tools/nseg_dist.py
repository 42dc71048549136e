"""Experiment (tools/): distribution of segments per batch by concurrency cap
on the C5 sweep (how many noise draws per batch the replay uses)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_18725_b200 import engine
from paper_2512_18725_b200.profiles import gen_synthetic_profiles
from paper_2512_18725_b200.sweep import c5_scenarios, lpt_order
table = gen_synthetic_profiles()
specs = lpt_order(c5_scenarios(table, 10000))
pipe = engine.ReplayPipeline(specs, table.arrays(), scale=1.5)
pipe.run(); torch.cuda.synchronize()
h = pipe.fetch()
caps = np.array([s["concurrency_cap"] if isinstance(s, dict) else s.concurrency_cap for s in specs]) if False else None
tot = {}
for s in range(len(specs)):
    v = pipe.scenario(h, s)
    cap = int(specs[s]["concurrency_cap"])
    ns = np.asarray(v["b_nseg"])
    tot.setdefault(cap, []).append(ns)
for cap, lst in tot.items():
    a = np.concatenate(lst)
    print(cap, len(a), np.bincount(a, minlength=10)[:12] / len(a))
