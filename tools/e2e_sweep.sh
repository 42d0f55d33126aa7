#!/usr/bin/env bash
# e2e at N GPUs for several PipelinedSteps layout SM budgets (VPX_PIPE_LAYOUT_SMS, 0 = all SMs)
N=$1; shift
for L in "$@"; do
  if [ "$N" = 1 ]; then VPX_PIPE_LAYOUT_SMS=$L timeout 600 python bench.py --no-cpu --no-aux > gpurun_out/e2e_${N}_$L.json 2> gpurun_out/e2e_${N}_$L.err
  else VPX_PIPE_LAYOUT_SMS=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29900+RANDOM%90)) bench.py --gpus $N --no-cpu > gpurun_out/e2e_${N}_$L.json 2> gpurun_out/e2e_${N}_$L.err; fi
  python - <<PY
import json
d=json.loads(open("gpurun_out/e2e_${N}_$L.json").read().strip().splitlines()[-1])
print("N=$N layout_sms=$L", round(d["value"],2), "e2e", round(d["e2e"]["value"],2), "i16", round(d["e2e_int16_host_input"]["value"],2))
PY
done
