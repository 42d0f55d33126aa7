#!/usr/bin/env bash
# Multi-GPU parity + scaling on one box (N = number of visible GPUs).
N=${1:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for cfg in "1x${N}x1x1 32 2 fp32" "2x$((N/2))x1x1 32 2 fp32" "1x$((N/2))x2x1 32 2 fp32" "1x${N}x1x1 128 2 tf32" "2x$((N/2))x1x1 128 2 tf32"; do
  timeout 300 $TR --master-port 29521 tools/check_dist.py $cfg 2>&1 | grep "check_dist\]"
done
# the NCCL send/recv halo path as well
VPX_NCCL_HALO=1 timeout 300 $TR --master-port 29521 tools/check_dist.py 1x$((N/2))x2x1 32 2 fp32 2>&1 | grep "check_dist\]"
timeout 600 $TR --master-port 29522 bench.py --gpus $N > gpurun_out/bench_${N}gpu.json 2> gpurun_out/bench_${N}gpu.err
tail -1 gpurun_out/bench_${N}gpu.err
python - <<PY
import json
l=json.loads(open('gpurun_out/bench_${N}gpu.json').read().strip().splitlines()[-1])
print("N=$N", l['value'], l['ms_per_step'], (l.get('e2e') or {}).get('value'))
PY
