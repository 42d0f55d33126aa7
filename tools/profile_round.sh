#!/usr/bin/env bash
# Round profiling recipe (run on a GPU box through gpurun, one GPU):
#   1. the bench line itself (no profiler)                  -> gpurun_out/<tag>_bench.json
#   2. ncu launch list of the same command (per-launch times) -> gpurun_out/<tag>_launches.csv
#   3. one `ncu --set full` capture of the top layers' kernels -> gpurun_out/<tag>_*.ncu-rep
# Each ncu step runs only after the plain command exited 0.
# Usage: tools/profile_round.sh <tag> [extra bench args]
set -u
TAG=${1:-r1}
shift || true
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-graph --no-aux $*"

timeout 900 python bench.py "$@" > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err || { echo "bench failed"; tail -5 $OUT/${TAG}_bench.err; exit 1; }
timeout 300 $BENCH > $OUT/${TAG}_plain.json 2> $OUT/${TAG}_plain.err || { echo "plain bench failed"; exit 1; }

timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/${TAG}_launches.csv $BENCH > $OUT/${TAG}_ncu_list.log 2>&1 || echo "launch list failed"

export VPX_NVTX=1
for grp in "c1.wgrad c1.fwd c2.wgrad" "c2.dgrad c2.fwd c3.dgrad c2_act.bwd"; do
  inc=""
  name=""
  for t in $grp; do inc="$inc --nvtx-include $t/"; name="${name}_${t//./}"; done
  timeout 1200 ncu --set full --clock-control none --import-source on --nvtx $inc -c 8 \
    -o $OUT/${TAG}${name} -f $BENCH > $OUT/${TAG}${name}.log 2>&1 || echo "ncu $grp failed"
done
echo done
