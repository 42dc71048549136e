"""Experiment (tools/): the host-buffer best-candidate call (intf_best_candidates_
host_sync, one launch) in a loop, for ncu / timing: per-call host time and the
kernel's device time by events."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_18725_b200 import engine  # noqa: E402
from paper_2512_18725_b200.profiles import gen_synthetic_profiles  # noqa: E402
from paper_2512_18725_b200.sweep import c2_decision_coefs  # noqa: E402

ta = gen_synthetic_profiles().arrays()
sc = engine.CandidateScorer(ta, cap=4, alpha=0.5)
hc = torch.tensor(c2_decision_coefs(32), dtype=torch.float64).pin_memory().numpy()
hb = torch.empty(2 * 32 * sc.E, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
scr = torch.empty(sc.best_scratch_elems(32) + sc.ws_elems, dtype=torch.float32, device="cuda")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for _ in range(20):
    sc.best_host_pipelined(hc, hb, scr, sync=True)
t0 = time.perf_counter()
for _ in range(n):
    sc.best_host_pipelined(hc, hb, scr, sync=True)
host_us = (time.perf_counter() - t0) / n * 1e6
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
sc.best_host_pipelined(hc, hb, scr)
e1.record()
torch.cuda.synchronize()
print(f"host call {host_us:.1f} us; one call's device time (launch to end, events) {e0.elapsed_time(e1) * 1e3:.1f} us")
