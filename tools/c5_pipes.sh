#!/bin/bash
# Experiment (tools/): C5 sweep time vs pipelines (INTF_BENCH_PIPES) at 20 timed steps
OUT=gpurun_out; mkdir -p $OUT
for P in ${@:-2 3 4}; do
  for rep in 1 2; do
  INTF_BENCH_PIPES=$P timeout 600 python bench.py --no-cpu --no-c4 > $OUT/bench_p$P.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$OUT/bench_p$P.json').read().strip().splitlines()[-1]); r=d['replay']
print('INTF_BENCH_PIPES=$P', r['steps_timed'], round(r['value']), round(r['ms_per_step'], 3), r['status_nonzero'])"
  done
done
