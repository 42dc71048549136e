#!/bin/bash
# Experiment (tools/): C5 sweep time vs noise draws precomputed per batch (INTF_NOISE_K)
OUT=gpurun_out; mkdir -p $OUT
for K in ${@:-3 4 5 6}; do

  for rep in 1 2; do
  INTF_NOISE_K=$K timeout 600 python bench.py --no-cpu --no-c4 > $OUT/bench_nk$K.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$OUT/bench_nk$K.json').read().strip().splitlines()[-1]); r=d['replay']
print('INTF_NOISE_K=$K', round(r['value']), round(r['ms_per_step'], 3), r['status_nonzero'], {k: round(v, 3) for k, v in r['stage_ms'].items()})"
  done
done
