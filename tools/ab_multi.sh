#!/usr/bin/env bash
# A/B of the N-GPU bench step on one box: tools/ab_multi.sh N "" "ENV=1" ...
N=$1; shift
i=0
for envs in "$@"; do
  for rep in 1 2; do
    env $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29950+RANDOM%40)) bench.py --gpus $N --no-cpu --no-e2e --no-aux > gpurun_out/abm_$i.json 2> gpurun_out/abm_$i.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/abm_$i.json").read().strip().splitlines()[-1])
print("N=$N [$envs] rep $rep", round(d["value"],2), round(d["ms_per_step"],4))
PY
  done
  i=$((i+1))
done
