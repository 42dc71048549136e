#!/bin/bash
# One gpurun session: GPU tests, smoke, bench, ncu launch list + top-kernel captures.
# usage (from the repo root, under gpurun):  bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > $OUT/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > $OUT/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_candidates -s 3 -c 1 -o $OUT/prof_cand_$TAG \
    python bench.py --steps 3 --warmup 3 --no-cpu > $OUT/ncu_cand_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 2 -c 1 -o $OUT/prof_replay_$TAG \
    python bench.py --steps 3 --warmup 3 --no-cpu > $OUT/ncu_replay_$TAG.log 2>&1
echo done
