#!/usr/bin/env bash
# bench.py at several GPU counts on one box (graph replay); prints value per N
for N in "$@"; do
  if [ "$N" = 1 ]; then timeout 400 python bench.py --no-cpu > gpurun_out/bench_1gpu.json 2> gpurun_out/bench_1gpu.err
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+N)) bench.py --gpus $N --no-cpu > gpurun_out/bench_${N}gpu.json 2> gpurun_out/bench_${N}gpu.err; fi
  python - <<PY
import json
l=json.loads(open('gpurun_out/bench_${N}gpu.json').read().strip().splitlines()[-1])
print("N=$N", round(l['value'],2), round(l['ms_per_step'],3), "e2e", round((l.get('e2e') or {}).get('value') or 0,2), l['step_mode'][:40], l['config'].get('halo'))
PY
done
