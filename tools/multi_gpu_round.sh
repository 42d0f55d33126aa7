#!/usr/bin/env bash
# Multi-GPU parity + scaling on one box (N = number of visible GPUs):
# tests/test_multigpu.py (halo bit-exactness, distributed step vs oracle,
# graph replays, stale memory), then the bench at N GPUs.
N=${1:-4}
timeout 2400 python -m pytest tests/test_multigpu.py -m gpu -q -s -p no:cacheprovider > gpurun_out/multigpu_${N}.log 2>&1
tail -3 gpurun_out/multigpu_${N}.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29522 \
  bench.py --gpus $N > gpurun_out/bench_${N}gpu.json 2> gpurun_out/bench_${N}gpu.err
tail -1 gpurun_out/bench_${N}gpu.err
