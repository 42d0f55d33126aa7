export VPX_NVTX=1
for R in c7.fwd c7.wgrad c6.dgrad c5.wgrad; do
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "$R/" -c 4 --csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-graph --no-aux > gpurun_out/small_$R.csv 2> gpurun_out/small_$R.err
done
