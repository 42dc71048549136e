"""Experiment (tools/): device time of each launch group of the C5 pipeline
(10^4 scenarios): arrivals, formation (+noise), replay kernel, SLO, features."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_18725_b200 import _abi, engine
from paper_2512_18725_b200.profiles import gen_synthetic_profiles
from paper_2512_18725_b200.sweep import c5_scenarios

table = gen_synthetic_profiles()
specs = c5_scenarios(table, 10000)
pipe = engine.ReplayPipeline(specs, table.arrays(), scale=1.5)
pipe.run()
L, s = pipe.lib, engine.stream_ptr()
bt, B = ctypes.byref(pipe.batch), ctypes.byref(pipe.B)
tab = ctypes.byref(pipe.dtable.struct)
for rep in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record()
    L.intf_generate_arrivals(bt, B, s)
    ev[1].record()
    L.intf_form_batches(bt, B, s)
    ev[2].record()
    L.intf_replay(bt, tab, B, s)  # formation + noise again, then the replay
    ev[3].record()
    pipe.run_slo_features(slo=True, features=False)
    ev[4].record()
    pipe.run_slo_features(slo=False, features=True)
    ev[5].record()
    torch.cuda.synchronize()
    names = ["arrivals", "formation+noise", "formation+noise+replay", "slo", "features"]
    print({n: round(ev[i].elapsed_time(ev[i + 1]), 3) for i, n in enumerate(names)})
