"""C2 step timing: materialised k_cand_step vs best-candidate k_cand_step<best>
(device-resident, PDL-chained) and the host-buffer best call."""
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
W = c2_decision_coefs(32)
sc = engine.CandidateScorer(ta, cap=4, alpha=0.5)
coefs = torch.tensor(W, device="cuda").contiguous()
outs = [sc.alloc(32), sc.alloc(32)]
bb = [sc.alloc_best(32), sc.alloc_best(32)]
K = 50
for mode in ("store", "best"):
    sc.pipeline_start(fused=True)
    for k in range(10):
        (sc.pipeline_step(coefs, outs[k & 1]) if mode == "store" else sc.best_step(coefs, bb[k & 1], bb[(k + 1) & 1]))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(K):
        (sc.pipeline_step(coefs, outs[k & 1]) if mode == "store" else sc.best_step(coefs, bb[k & 1], bb[(k + 1) & 1]))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"{mode}: {1e3 * ms:.2f} us/step  {64e6 * 0.9996 / (ms / 1e3):.3e} predictions/s")
hc = torch.tensor(W).pin_memory().numpy()
hb = torch.empty(2 * 32 * sc.E, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
scr = torch.empty(sc.best_scratch_elems(32), dtype=torch.float32, device="cuda")
for _ in range(10):
    sc.best_host(hc, hb, scr)
    torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(K):
    sc.best_host(hc, hb, scr)
    torch.cuda.synchronize()
print(f"best_host e2e: {1e6 * (time.perf_counter() - t0) / K:.1f} us/call")
scr2 = torch.empty(sc.best_scratch_elems(32) + sc.ws_elems, dtype=torch.float32, device="cuda")
for _ in range(10):
    sc.best_host_pipelined(hc, hb, scr2)
    torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(K):
    sc.best_host_pipelined(hc, hb, scr2)
    torch.cuda.synchronize()
print(f"best_host_pipelined e2e: {1e6 * (time.perf_counter() - t0) / K:.1f} us/call")
