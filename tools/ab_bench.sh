#!/usr/bin/env bash
# A/B the bench step on one box: each argument is an env assignment list
# ("" = default), e.g. tools/ab_bench.sh "" "VPX_NO_PREPACK=1"
i=0
for envs in "$@"; do
  for rep in 1 2; do
    env $envs timeout 300 python bench.py --no-aux --no-e2e --no-cpu --steps 20 > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/ab_$i.json").read().strip().splitlines()[-1])
print("[$envs] rep $rep", round(d["value"],2), round(d["ms_per_step"],4))
PY
  done
  i=$((i+1))
done
