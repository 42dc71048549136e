"""Experiment (tools/): C4 busy-period jobs -- distribution of job lengths
after the plan, and pass 1's time with the todo list in plan (time) order vs
longest-first (LPT by batches)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_18725_b200 import engine  # noqa: E402
from paper_2512_18725_b200.sweep import c4_scenario, table16  # noqa: E402

t16, arch = table16()
spec = c4_scenario(t16, arch, n_requests=1e6, seed=1)
pipe = engine.ReplayPipeline([spec], t16.arrays(), scale=1.5)
engine.replay_segmented(pipe, min_len=96, passes=4)  # sets up pipe._jobs
torch.cuda.synchronize()
L, st = pipe.lib, engine.stream_ptr()
bt, B = ctypes.byref(pipe.batch), ctypes.byref(pipe.B)
J = ctypes.byref(pipe._jobs.J)
tab = ctypes.byref(pipe.dtable.struct)
t = pipe._jobs.t
for mode in ("plan order", "LPT", "plan order", "LPT"):
    L.intf_generate_arrivals(bt, B, st)
    L.intf_form_batches(bt, B, st)
    L.intf_jobs_plan(bt, tab, B, J, st)
    torch.cuda.synchronize()
    n = int(t["todo_count"][0].item())
    todo = t["todo"][:n]
    ln = (t["hi"] - t["lo"])[todo.long()]
    if mode == "LPT":
        t["todo"][:n] = todo[torch.argsort(ln, descending=True)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.intf_jobs_replay(bt, tab, B, J, n, st)
    e1.record()
    torch.cuda.synchronize()
    lc = ln.cpu().numpy()
    print(f"{mode:10s}: pass 1 {e0.elapsed_time(e1):.3f} ms over {n} jobs; batches per job min {lc.min()} "
          f"median {int(np.median(lc))} p99 {int(np.percentile(lc, 99))} max {lc.max()} sum {lc.sum()}")
