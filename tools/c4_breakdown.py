"""Experiment (tools/): stage times of the C4 busy-period-sharded replay."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_18725_b200 import _abi, engine
from paper_2512_18725_b200.sweep import c4_scenario, table16

t16, arch = table16()
spec = c4_scenario(t16, arch, n_requests=1e6, seed=1)
pipe = engine.ReplayPipeline([spec], t16.arrays(), scale=1.2)
slow = float(os.environ.get("SLOW", "2.0"))
ml = int(os.environ.get("MIN_LEN", "16"))
engine.replay_segmented(pipe, slow=slow, min_len=ml)
torch.cuda.synchronize()
L, st = pipe.lib, engine.stream_ptr()
bt, B = ctypes.byref(pipe.batch), ctypes.byref(pipe.B)
J = ctypes.byref(pipe._jobs.J)
tab = ctypes.byref(pipe.dtable.struct)
ev = []


def mark(name):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    ev.append((name, e))


mark("start")
L.intf_generate_arrivals(bt, B, st)
mark("arrivals")
L.intf_form_batches(bt, B, st)
mark("formation+noise")
L.intf_jobs_plan(bt, tab, B, J, st)
mark("plan")
it = 0
while True:
    n = int(pipe._jobs.t["todo_count"][0].item())
    if n == 0:
        break
    it += 1
    L.intf_jobs_replay(bt, tab, B, J, n, st)
    mark(f"replay{it}({n})")
    L.intf_jobs_verify(bt, B, J, st)
    mark(f"verify{it}")
pipe.run_slo_features(slo=True, features=False)
mark("slo")
pipe.run_slo_features(slo=False, features=True)
mark("features")
torch.cuda.synchronize()
tot = ev[0][1].elapsed_time(ev[-1][1])
print(f"slow={slow} min_len={ml} total {tot:.2f} ms")
for (a, ea), (b, eb) in zip(ev, ev[1:]):
    print(f"  {b:>24s} {ea.elapsed_time(eb):8.3f} ms")
