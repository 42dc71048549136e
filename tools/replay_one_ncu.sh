#!/bin/bash
# ncu source-level capture of the longest cap-2 C5 scenario replayed alone (one warp: the serial chain)
# usage (under gpurun): bash tools/replay_one_ncu.sh TAG
TAG=${1:-one}
mkdir -p gpurun_out
MIN_CAP=2 timeout 400 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --clock-control none \
  --import-source on -k regex:k_replay_warp -s 3 -c 1 -o gpurun_out/prof_$TAG python tools/replay_one.py > gpurun_out/ncu_$TAG.log 2>&1
