"""Experiment (tools/): the C4 arrivals stage alone -- k_gen_gaps, the
cumulative-sum kernels (k_bin_*, or k_scan_gaps when built with
INTF_SCAN_SEQ=1), k_fill_gaps -- timed with events, plus the binade scan's
chunk classes per long model (clean / sequential / run heads)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_18725_b200 import engine
from paper_2512_18725_b200.sweep import c4_scenario, table16

t16, arch = table16()
spec = c4_scenario(t16, arch, n_requests=1e6, seed=1)
pipe = engine.ReplayPipeline([spec], t16.arrays(), scale=1.2)
L, st = pipe.lib, engine.stream_ptr()
bt, B = ctypes.byref(pipe.batch), ctypes.byref(pipe.B)
for _ in range(3):
    L.intf_generate_arrivals(bt, B, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    L.intf_generate_arrivals(bt, B, st)
e1.record()
torch.cuda.synchronize()
print(f"arrivals stage {e0.elapsed_time(e1) / 10:.3f} ms")
mb = pipe.t["mb_t"].cpu().numpy()
for g in range(pipe.pb.n_models):
    m = pipe.pb.models[g]
    cap = m.list_cap
    if cap < 4096 or m.rate_rps == 0:
        continue
    n32 = cap // 32
    seg = mb[m.list_off: m.list_off + cap]
    code = seg[4 * n32: 4 * n32 + (n32 + 1) // 2].view(np.int32)[:n32]
    clean = code >= 0
    heads = (code >= 0) & ((code & (1 << 20)) != 0)
    print(f"model {g}: cap {cap} chunks {n32} clean {clean.sum()} sequential {(~clean).sum()} runs {heads.sum()}")
