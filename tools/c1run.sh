mkdir -p gpurun_out/$1
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_guards.py tests/test_gpu_slabs512.py -x -q -k "first_block or c1 or slab" > gpurun_out/$1/t.log 2>&1; tail -3 gpurun_out/$1/t.log
python bench.py --no-aux --no-e2e > gpurun_out/$1/bench.json 2> gpurun_out/$1/bench.err
python - <<PY
import json
d=json.loads(open("gpurun_out/$1/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"])
for k in ["c1.fwd","c1.wgrad"]: print(k, d["kernels"][k])
PY
