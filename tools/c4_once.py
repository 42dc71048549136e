"""One C4 trace (10^6 requests, busy-period-sharded replay + SLO) for
profiling: `ncu ... python tools/c4_once.py`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_18725_b200 import engine  # noqa: E402
from paper_2512_18725_b200.sweep import c4_scenario, table16  # noqa: E402

t16, arch = table16()
pipe = engine.ReplayPipeline([c4_scenario(t16, arch, n_requests=1e6, seed=1)], t16.arrays(), scale=1.5)
st = engine.replay_segmented(pipe, min_len=32, passes=2)
torch.cuda.synchronize()
print("status", int(pipe.status()[0]), {k: st[k] for k in st if k.startswith("jobs")})
