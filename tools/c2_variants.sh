#!/bin/bash
# Experiment (tools/): each build/variants/*.so on the C2 best step and the host call
cd "$(dirname "$0")/.."
L=paper_2512_18725_b200/_lib/libintfsim_b200.so
cp $L /tmp/lib_orig.so
for v in build/variants/*.so build/variants/*.so; do
  cp "$v" $L; echo "== $(basename $v .so)"
  python tools/c2_best_timing.py 2>&1 | grep -E "^best:|pipelined"
  python tools/c2_host_once.py 1000
done
cp /tmp/lib_orig.so $L
