#!/bin/bash
# quick gpurun: GPU tests, the longest cap-2 C5 scenario alone (twice), bench without the CPU legs
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gq_tests.log 2>&1; echo rc=$? >> gpurun_out/gq_tests.log
MIN_CAP=2 python tools/replay_one.py > gpurun_out/gq_one.log 2>&1
MIN_CAP=2 python tools/replay_one.py >> gpurun_out/gq_one.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/gq_bench.json 2> gpurun_out/gq_bench.err
