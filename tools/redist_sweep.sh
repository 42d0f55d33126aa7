#!/usr/bin/env bash
# bench.py at N GPUs for several redistribution points (graph replay)
N=$1; shift
for r in "$@"; do
  arg=""; [ "$r" != default ] && arg="--redistribute-before $r"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700+RANDOM%200)) \
    bench.py --gpus $N --no-cpu --no-e2e $arg > gpurun_out/rd_${N}_$r.json 2> gpurun_out/rd_${N}_$r.err
  python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/rd_${N}_$r.json").read().strip().splitlines()[-1])
    print("N=$N redist $r", round(d["value"],2), round(d["ms_per_step"],4), d["config"]["redistribute_before"])
except Exception as e:
    print("N=$N redist $r failed", e)
PY
done
