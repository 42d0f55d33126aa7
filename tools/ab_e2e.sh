#!/usr/bin/env bash
# A/B of the bench line (value and e2e) on one box: each argument is an env list ("" = default)
i=0
for envs in "$@"; do
  for rep in 1 2; do
    env $envs timeout 400 python bench.py --no-aux --no-cpu --steps 20 > gpurun_out/abe_$i.json 2> gpurun_out/abe_$i.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/abe_$i.json").read().strip().splitlines()[-1])
print("[$envs] rep $rep", round(d["value"],2), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"],2), "i16", round(d["e2e_int16_host_input"]["value"],2))
PY
  done
  i=$((i+1))
done
