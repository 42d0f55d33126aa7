set -u
O=gpurun_out/prof4
mkdir -p $O
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-graph --no-aux"
timeout 300 $BENCH > $O/plain.json 2> $O/plain.err || { echo "plain failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $BENCH > $O/ncu_list.log 2>&1 || echo "launch list failed"
export VPX_NVTX=1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "c1.fwd/" --nvtx-include "c1.wgrad/" -k "regex:c1_" -c 2 -o $O/c1 -f $BENCH > $O/c1.log 2>&1 || echo "ncu c1 failed"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "c2.wgrad/" --nvtx-include "c2.dgrad/" --nvtx-include "c3.dgrad/" -k "regex:wgrad_ut|rowh|rowwin" -c 3 -o $O/c23 -f $BENCH > $O/c23.log 2>&1 || echo "ncu c23 failed"
echo done
