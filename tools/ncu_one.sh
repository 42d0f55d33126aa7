#!/usr/bin/env bash
# One `ncu --set full` capture of the launches inside one NVTX layer range of
# the eager bench step (single GPU).  Usage: tools/ncu_one.sh <tag> <layer.pass> [count] [kernel regex]
set -u
TAG=$1; RANGE=$2; CNT=${3:-1}; KRE=${4:-.}
mkdir -p gpurun_out
export VPX_NVTX=1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$RANGE/" -k "regex:$KRE" -c "$CNT" \
  -o gpurun_out/${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-graph --no-aux \
  > gpurun_out/${TAG}.log 2>&1 || { echo "ncu failed"; tail -20 gpurun_out/${TAG}.log; exit 1; }
echo "captured gpurun_out/${TAG}.ncu-rep"
