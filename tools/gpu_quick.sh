#!/bin/bash
# quick gpurun: GPU tests + bench (+ optional ncu --set full of kernels matching each regex)
# usage: bash tools/gpu_quick.sh TAG [regex ...]
TAG=${1:-q}; shift
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
for K in "$@"; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $OUT/prof_${TAG}_$K \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-c4 > $OUT/ncu_${TAG}_$K.log 2>&1
done
echo done
