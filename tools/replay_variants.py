"""Experiment (tools/): time the C5 replay stage of whatever library is in
place (build/variants/*.so swapped in by tools/replay_variants.sh) and print a
checksum of the replay outputs, so tuning variants are compared on speed AND
on identical results.  usage: python tools/replay_variants.py NAME"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_18725_b200 import engine  # noqa: E402
from paper_2512_18725_b200.profiles import gen_synthetic_profiles  # noqa: E402
from paper_2512_18725_b200.sweep import c5_scenarios, lpt_order  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "current"
table = gen_synthetic_profiles()
pipe = engine.ReplayPipeline(lpt_order(c5_scenarios(table, 10000)), table.arrays(), scale=1.5)
stream = torch.cuda.current_stream()
pipe.run()
torch.cuda.synchronize()
h = pipe.fetch()
dig = hashlib.sha256()
for k in sorted(h):
    v = h[k]
    if isinstance(v, np.ndarray):
        dig.update(k.encode())
        dig.update(np.ascontiguousarray(v).tobytes())
times = [bench.replay_stage_times(pipe, stream) for _ in range(7)]
med = {k: float(np.median([t[k] for t in times])) for k in ("arrivals", "replay", "slo", "features")}
print(json.dumps({"variant": name, "replay_ms": med["replay"], "stages": med, "status": int((pipe.status() != 0).sum()),
                  "sha": dig.hexdigest()[:16]}))
