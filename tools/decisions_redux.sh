#!/bin/bash
# Experiment (tools/): decision argmin by packed 64-bit shuffle min (default) vs redux.sync
python tools/decisions_timing.py
INTF_NVCC_EXTRA=-DINTF_DECISION_REDUX python -c "from paper_2512_18725_b200 import build; build.build(force=True)" && echo "--- redux.sync" && python tools/decisions_timing.py
