#!/bin/bash
# Experiment (tools/): each build/variants/*.so on the C5 stage times
# (tools/replay_variants.py) and the pipelined steady-state sweep (tools/c5_sens.py)
cd "$(dirname "$0")/.."
L=paper_2512_18725_b200/_lib/libintfsim_b200.so
cp $L /tmp/lib_orig.so
for v in build/variants/*.so; do
  cp "$v" $L
  n=$(basename "$v" .so)
  timeout 300 python tools/replay_variants.py "$n" 2>&1 | tail -1
  echo "$n $(timeout 300 python tools/c5_sens.py 2>&1 | tail -1)"
done
cp /tmp/lib_orig.so $L
