#!/bin/bash
# Experiment (tools/): time every build/variants/*.so on the C5 replay stage
# (run on the GPU box: tools/build_variants.sh first, here)
cd "$(dirname "$0")/.."
L=paper_2512_18725_b200/_lib/libintfsim_b200.so
cp $L /tmp/lib_orig.so
for v in build/variants/*.so; do
  cp "$v" $L
  timeout 300 python tools/replay_variants.py "$(basename "$v" .so)" 2>&1 | tail -1
done
cp /tmp/lib_orig.so $L
