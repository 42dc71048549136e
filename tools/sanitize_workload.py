"""Small runs of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck): the smoke (bundled trace replay + features + a cap-3
candidate step), a 2x10^5-request C4 trace (long-list arrivals / formation /
busy-period jobs / grid SLO), a 256-scenario C5 sweep with the per-scenario
evaluation, the best-candidate step, the windowed OLS (TMA), the
RLS / SGD / drift paths, the one-launch host best-candidate call and the
SLO edge cases (ties above the warp-rank limit, > 2,048 records)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.smoke()
import paper_2512_18725_b200 as p  # noqa: E402
from paper_2512_18725_b200 import _abi, engine, experiments as ex  # noqa: E402
from paper_2512_18725_b200.sweep import c2_decision_coefs, c4_scenario, c5_scenarios, lpt_order, table16  # noqa: E402

t16, arch = table16()
pipe = engine.ReplayPipeline([c4_scenario(t16, arch, n_requests=2e5)], t16.arrays(), scale=1.5)
st = engine.replay_segmented(pipe, passes=4)
print("c4 2e5", st, int(pipe.status()[0]))
table = p.gen_synthetic_profiles()
preds = [_abi.Predictor(ewma=0, alpha=1.0, w=(0.0,) * 7), _abi.Predictor(ewma=1, alpha=0.5, w=(0.0,) * 7)]
pp = engine.ReplayPipeline(lpt_order(c5_scenarios(table, 256)), table.arrays(), preds=preds, scale=1.5,
                           evaluate=(0, 1, 0.99))
pp.run()
torch.cuda.synchronize()
print("c5 256", int((pp.status() != 0).sum()), int((pp.eval_status.cpu().numpy()[:256] & 1).sum()))
sc = engine.CandidateScorer(table.arrays(), cap=3, alpha=0.5)
W = torch.tensor(c2_decision_coefs(8), device="cuda").contiguous()
bb = [sc.alloc_best(8) for _ in range(2)]
sc.pipeline_start(fused=True)
sc.best_step(W, bb[0], bb[1])
torch.cuda.synchronize()
sc4 = engine.CandidateScorer(table.arrays(), cap=4, alpha=0.5)
sc4.prepare_decisions()
rank, own = sc4.dispatch_decisions(pp)
best, chosen = sc4.score_decisions(W[0].contiguous(), rank, own)
torch.cuda.synchronize()
print("decisions", int((rank >= 0).sum()))
X = np.random.default_rng(0).uniform(0, 1, size=(4096, 6))
y = X @ np.arange(1, 7) + 1.0
print("ols windows", len(p.predict.fit_ols_windows(X, y, 64)))
cells = ex.drift_experiment(ex.default_drift_base(table, 0), table)
print("drift", len(cells))
# the one-launch host call (pinned keys written by the last block, completion word) and the copy path
hc = torch.tensor(c2_decision_coefs(8), dtype=torch.float64).pin_memory().numpy()
hb = torch.empty(2 * 8 * sc.E, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
scr = torch.empty(sc.best_scratch_elems(8) + sc.ws_elems, dtype=torch.float32, device="cuda")
for _ in range(3):
    sc.best_host_pipelined(hc, hb, scr, sync=True)
sc.best_host_pipelined(hc, np.zeros_like(hb), scr, sync=True)
print("host calls", int(hb[0] >> 32))
# SLO edges: tied latencies beyond the warp-rank limit, > 2,048 records (crafted arrivals)
bursts = np.repeat(np.arange(0.0, 1000.0, 14.0), 35)
t_arr = np.sort(np.concatenate([bursts, np.linspace(1.0, 999.0, 120)]))
m_arr = np.zeros(len(t_arr), dtype=np.int32)
m_arr[np.isin(t_arr, bursts, invert=True)] = 1
spec = {"name": "ties", "duration_s": 1.0, "batching_window_ms": 2.0, "max_batch_size": 64, "concurrency_cap": 3,
        "seed": 0, "colocation_mode": "static", "ewma_alpha": 1.0,
        "oracle": {"beta_l2": 1.0, "beta_dram": 1.5, "beta_sm": 0.5, "noise_sigma": 0.05, "seed": 0},
        "deployed": [{"model_id": m, "arrival_rate_rps": 100.0, "slo_ms": 100.0} for m in t16.models()[:2]]}
pt, _ = engine.run_batch([spec], t16.arrays(), arrivals=[(t_arr, m_arr)], warmup_fraction=0.3)
print("slo edges", int(pt.status()[0]))
