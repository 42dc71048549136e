#!/bin/bash
# Experiment (tools/): RLS update latency -- exact divisions vs reciprocal multiplies
python tools/rls_latency.py
INTF_NVCC_EXTRA=-DINTF_RLS_RECIP python -c "from paper_2512_18725_b200 import build; build.build(force=True)" && echo "--- INTF_RLS_RECIP" && python tools/rls_latency.py
