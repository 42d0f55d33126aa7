#!/usr/bin/env bash
# Round-end validation on one 4-GPU box: the whole -m gpu suite (multi-GPU
# cases included), smoke(), bench at 1/2/4 GPUs, the reference arm, U-Net.
# Usage: tools/final_round.sh <outdir under gpurun_out>
O=gpurun_out/${1:-final}
mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_1gpu.json 2> $O/bench_1gpu.err; tail -c 300 $O/bench_1gpu.json; echo
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29800+N)) \
    bench.py --gpus $N > $O/bench_${N}gpu.json 2> $O/bench_${N}gpu.err
done
timeout 900 python bench.py --impl reference > $O/ref_1gpu.json 2> $O/ref_1gpu.err
timeout 600 python bench.py --net unet --no-cpu > $O/bench_unet_1gpu.json 2> $O/bench_unet_1gpu.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 \
  bench.py --gpus 4 --net unet --no-cpu > $O/bench_unet_4gpu.json 2> $O/bench_unet_4gpu.err
python - <<PY
import json
for f in ["bench_1gpu","bench_2gpu","bench_4gpu","ref_1gpu","bench_unet_1gpu","bench_unet_4gpu"]:
    try:
        d=json.loads(open("$O/"+f+".json").read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), (d.get("roofline") or {}).get("frac"))
    except Exception as e:
        print(f, "failed", e)
PY
