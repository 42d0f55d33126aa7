#!/usr/bin/env bash
# Launch list of the eager bench step + ncu --set full of c2 fwd / c2 dgrad / c3 fwd at HEAD (one GPU)
O=gpurun_out/prof8; mkdir -p $O
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-graph --no-aux"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $BENCH > $O/ncu_list.log 2>&1 || echo "launch list failed"
export VPX_NVTX=1
B1="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-graph --no-aux"
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "c2.fwd/" --nvtx-include "c2.dgrad/" --nvtx-include "c3.fwd/" -k "regex:rowh|rowwin" -c 3 -o $O/c23 -f $B1 > $O/c23.log 2>&1 || echo "ncu failed"
echo done
