#!/usr/bin/env bash
# PDL A/B on one box: deep-layer passes (graph of 50) and the 1-GPU bench step, with and without VPX_NO_PDL
set -x
timeout 300 python -m pytest -q -x -m gpu tests/test_gpu_kernels.py tests/test_gpu_engine.py 2>&1 | tail -3
timeout 120 python tools/small_pass.py
VPX_NO_PDL=1 timeout 120 python tools/small_pass.py
bash tools/ab_bench.sh "" "VPX_NO_PDL=1" ""
