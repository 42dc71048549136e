#!/bin/bash
# Experiment (tools/): C5 sweep time vs INTF_LONG_LIST (lists at least this
# long form batches by pointer doubling instead of the warp walk); each
# variant rebuilt, checked against the goldens, and benched.
OUT=gpurun_out; mkdir -p $OUT
for N in ${@:-4096 256 64 1}; do
  INTF_NVCC_EXTRA="-DINTF_LONG_LIST=$N" python -c "from paper_2512_18725_b200 import build; build.build(force=True)" > $OUT/build_ll$N.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_replay.py tests/test_gpu_api.py -q -m gpu 2>&1 | tail -1
  timeout 600 python bench.py --no-cpu --no-c4 > $OUT/bench_ll$N.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$OUT/bench_ll$N.json').read().strip().splitlines()[-1]); r=d['replay']
print('INTF_LONG_LIST=$N', round(r['value']), round(r['ms_per_step'], 3), r['status_nonzero'], r['stage_ms'])"
done
python -c "from paper_2512_18725_b200 import build; build.build(force=True)" > /dev/null 2>&1
