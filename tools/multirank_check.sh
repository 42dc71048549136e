#!/bin/bash
# Plumbing check of the N > 1 bench path on a 1-GPU box: 2 ranks share cuda:0
# over gloo (numbers meaningless), then the reference arm under torchrun.
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-cpu > $OUT/mr_bench.json 2> $OUT/mr_bench.err; echo "rc=$?" >> $OUT/mr_bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $OUT/mr_ref.json 2> $OUT/mr_ref.err; echo "rc=$?" >> $OUT/mr_ref.err
