export VPX_NVTX=1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "e1c1.wgrad/" -k "regex:c1k3" -c 1 -o gpurun_out/e1c1w -f python bench.py --net unet --steps 1 --warmup 3 --no-cpu --no-e2e --no-graph --no-aux > gpurun_out/e1c1w.log 2>&1 || echo fail
