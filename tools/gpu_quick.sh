#!/bin/bash
# quick gpurun: GPU tests + bench (+ optional ncu of one kernel regex)
TAG=${1:-q}
KREGEX=${2:-}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
if [ -n "$KREGEX" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 3 -c 1 -o $OUT/prof_${TAG} \
    python bench.py --steps 3 --warmup 3 --no-cpu > $OUT/ncu_$TAG.log 2>&1
fi
echo done
