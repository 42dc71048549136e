#!/bin/bash
# Experiment (tools/): C4 back-to-back traces vs pipelines (INTF_BENCH_C4_PIPES)
OUT=gpurun_out; mkdir -p $OUT
for P in ${@:-2 3}; do
  for rep in 1 2; do
  INTF_BENCH_C4_PIPES=$P timeout 600 python bench.py --no-cpu > $OUT/bench_c4p$P.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$OUT/bench_c4p$P.json').read().strip().splitlines()[-1]); c=d['long_trace']
print('INTF_BENCH_C4_PIPES=$P', round(c['ms_per_trace'], 3), c['pipelined'])"
  done
done
