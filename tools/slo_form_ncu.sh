#!/bin/bash
# Experiment (tools/): source-level ncu of the C5 formation + SLO kernels
# (k_slo, k_form_models, k_merge_batches) from one 10^4-scenario sweep
# usage (under gpurun): bash tools/slo_form_ncu.sh TAG
TAG=${1:-sf}
mkdir -p gpurun_out
for K in ${KERNELS:-k_slo k_form_models k_merge_batches}; do
  timeout 300 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --section MemoryWorkloadAnalysis \
    --clock-control none --import-source on -k regex:"^$K\$|::$K\(" -c 1 -o gpurun_out/prof_${TAG}_$K \
    env C5_ONCE_PLAIN=1 python tools/c5_once.py > gpurun_out/ncu_${TAG}_$K.log 2>&1
done
