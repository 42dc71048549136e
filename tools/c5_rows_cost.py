"""C5 bench step with / without the per-scenario row build (SweepRows)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_18725_b200 import _abi, engine  # noqa: E402
from paper_2512_18725_b200.distributed import SweepRows  # noqa: E402
from paper_2512_18725_b200.profiles import gen_synthetic_profiles  # noqa: E402
from paper_2512_18725_b200.sweep import c5_scenarios, lpt_order  # noqa: E402

table = gen_synthetic_profiles()
specs = lpt_order(c5_scenarios(table, 10000))
preds = [_abi.Predictor(ewma=0, alpha=1.0, w=(0.0,) * 7), _abi.Predictor(ewma=1, alpha=0.5, w=(0.0,) * 7)]
pipes = [engine.ReplayPipeline(specs, table.arrays(), preds=preds, scale=1.5, evaluate=(0, 1, 0.99)) for _ in range(3)]
rows = [SweepRows(p) for p in pipes]
for p in pipes:
    p.run()
torch.cuda.synchronize()
streams = [torch.cuda.Stream() for _ in pipes]
for build in (False, True, False, True):
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for s in streams:
        s.wait_stream(cur)
    for k in range(20):
        with torch.cuda.stream(streams[k % 3]):
            pipes[k % 3].run()
            if build:
                rows[k % 3].build()
    host = time.perf_counter() - t0
    for s in streams:
        cur.wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    print(f"rows.build {build}: {e0.elapsed_time(e1) / 20:.3f} ms/step (host enqueue {1e3 * host / 20:.3f} ms/step)")
