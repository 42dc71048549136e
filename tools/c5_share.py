"""C5 strong-scaling share on ONE GPU: rank r's LPT share of the fixed 10^4
sweep at world W, replayed on P pipelines (consecutive sweeps in flight),
vs the whole sweep: is the per-GPU time near (whole sweep) / W?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_18725_b200 import _abi, engine  # noqa: E402
from paper_2512_18725_b200.distributed import lpt_shards  # noqa: E402
from paper_2512_18725_b200.profiles import gen_synthetic_profiles  # noqa: E402
from paper_2512_18725_b200.sweep import c5_scenarios, expected_requests  # noqa: E402

table = gen_synthetic_profiles()
ta = table.arrays()
specs_all = c5_scenarios(table, 10000)
w = [expected_requests(s) for s in specs_all]
preds = [_abi.Predictor(ewma=0, alpha=1.0, w=(0.0,) * 7), _abi.Predictor(ewma=1, alpha=0.5, w=(0.0,) * 7)]


def sweep_ms(specs, n_pipes, steps):
    pipes = [engine.ReplayPipeline(specs, ta, preds=preds, scale=1.5, evaluate=(0, 1, 0.99)) for _ in range(n_pipes)]
    for p in pipes:
        p.run()
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in pipes]
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_stream(cur)
    for k in range(steps):
        with torch.cuda.stream(streams[k % n_pipes]):
            pipes[k % n_pipes].run()
    for s in streams:
        cur.wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


full = sweep_ms(specs_all, 3, 12)
print(f"whole 10^4 sweep, 3 pipelines: {full:.3f} ms/sweep")
for world in (2, 4, 8):
    sh = lpt_shards(w, world)[0]
    specs = [specs_all[i] for i in sh]
    for n_pipes in sorted({3 * world, 4 * world, 2 * world}):
        ms = sweep_ms(specs, n_pipes, max(4 * n_pipes, 24))
        print(f"world {world}: rank-0 share {len(specs)} scenarios, {n_pipes} pipelines: {ms:.3f} ms/sweep "
              f"= {ms / (full / world):.2f} x (whole / {world})")
