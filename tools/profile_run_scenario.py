"""cProfile of run_scenario (C1 e2e) on the bundled trace."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18725_b200 as p  # noqa: E402
from paper_2512_18725_b200.sweep import BUNDLED_SEED7  # noqa: E402
from paper_2512_18725_b200.workload import scenario_from_dict  # noqa: E402

table = p.gen_synthetic_profiles()
spec = scenario_from_dict(BUNDLED_SEED7)
for _ in range(3):
    p.run_scenario(spec, table)
t0 = time.perf_counter()
for _ in range(10):
    p.run_scenario(spec, table)
print(f"run_scenario: {(time.perf_counter() - t0) * 100:.2f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    p.run_scenario(spec, table)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
