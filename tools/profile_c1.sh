#!/usr/bin/env bash
# ncu --set full of the two first-block kernels (c1 forward, c1 filter gradient), one GPU
O=gpurun_out/prof6; mkdir -p $O
BENCH="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-graph --no-aux"
export VPX_NVTX=1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "c1.fwd/" -k "regex:c1_fwd_pool" -c 1 -o $O/c1fwd -f $BENCH > $O/c1fwd.log 2>&1 || echo "c1fwd failed"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "c1.wgrad/" -k "regex:c1_pooled" -c 1 -o $O/c1wgrad -f $BENCH > $O/c1wgrad.log 2>&1 || echo "c1wgrad failed"
echo done
