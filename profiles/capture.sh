#!/bin/bash
# Round-1 profiling recipe (run under gpurun from the repo root; outputs in gpurun_out/):
#   a launch list (every kernel of one eager analysis: time + DRAM bytes) and one
#   `ncu --set full` capture of the top kernels (roofline `traffic`, stall reasons).
#   usage: bash profiles/capture.sh <workload> "<kernel regex>" <count>
set -u
W=${1:-c5}
K=${2:-"k_rs_down_tma|k_rs_onesweep<unsigned int>|k_access|k_acc_keys"}
C=${3:-3}
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
  python profiles/run_one.py --workload $W --repeat 1 > gpurun_out/ncu_l_$W.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c $C \
  -o gpurun_out/full_$W python profiles/run_one.py --workload $W --repeat 1 > gpurun_out/ncu_f_$W.log 2>&1
for f in gpurun_out/ncu_l_$W.log gpurun_out/ncu_f_$W.log; do tail -n 1 $f; done
