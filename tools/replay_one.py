"""Experiment (tools/): the longest C5 scenario (of the first 10^4) replayed
alone -- one warp on the GPU, i.e. the replay's serial critical path.  For
`ncu -k regex:k_replay_warp`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_18725_b200 import engine
from paper_2512_18725_b200.profiles import gen_synthetic_profiles
from paper_2512_18725_b200.sweep import c5_scenarios

table = gen_synthetic_profiles()
specs = c5_scenarios(table, 10000)
pipe = engine.ReplayPipeline(specs, table.arrays(), scale=1.5)
pipe.run()
nb = pipe.t["n_batches"][: pipe.pb.n_scen].cpu().numpy()
caps = [sp["concurrency_cap"] for sp in specs]
min_cap = int(os.environ.get("MIN_CAP", "1"))
i = max((k for k in range(len(specs)) if caps[k] >= min_cap), key=lambda k: nb[k])
one = engine.ReplayPipeline([specs[i]], table.arrays(), scale=1.5)
for _ in range(3):
    one.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
one.run()
e1.record()
torch.cuda.synchronize()
print(f"scenario {i}: {int(nb[i])} batches, cap {specs[i]['concurrency_cap']}, {e0.elapsed_time(e1):.3f} ms")
