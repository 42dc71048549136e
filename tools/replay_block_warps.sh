#!/bin/bash
# Experiment (tools/): C5 sweep and C4 trace time vs warps per replay block (INTF_REPLAY_WARPS = INTF_JOB_WARPS;
# 12 resident warps per SM in every variant).  A persistent block holds its
# registers until its LAST warp ends, so with 4-warp blocks one long scenario
# keeps three finished warps' slots from the next sweep's kernels.
OUT=gpurun_out; mkdir -p $OUT
for N in ${@:-4 2 1}; do
  INTF_NVCC_EXTRA="-DINTF_REPLAY_WARPS=$N -DINTF_JOB_WARPS=$N" python -c "from paper_2512_18725_b200 import build; build.build(force=True)" > $OUT/build_rw$N.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_replay.py tests/test_gpu_api.py tests/test_gpu_segmented.py -q -m gpu 2>&1 | tail -1
  for rep in 1 2; do
  timeout 600 python bench.py --no-cpu > $OUT/bench_rw$N.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$OUT/bench_rw$N.json').read().strip().splitlines()[-1]); r=d['replay']; c=d['long_trace']
print('INTF_REPLAY_WARPS=$N', round(r['value']), round(r['ms_per_step'], 3), r['status_nonzero'], {k: round(v, 3) for k, v in r['stage_ms'].items()}, 'C4', round(c['ms_per_trace'], 3), round(c['pipelined']['ms_per_trace'], 3))"
  done
done
python -c "from paper_2512_18725_b200 import build; build.build(force=True)" > /dev/null 2>&1
