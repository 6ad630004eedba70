#!/bin/bash
# Round-1 profiling recipe (run under gpurun from the repo root; outputs in gpurun_out/):
#   launch lists (every kernel of one eager analysis: time + DRAM bytes) for C2 and C5,
#   and one `ncu --set full` capture of the top kernels for the roofline `traffic` field.
set -u
W=${1:-c5}
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
  python profiles/run_one.py --workload $W --repeat 1 > gpurun_out/ncu_l_$W.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_rs_down|k_rs_onesweep<unsigned int>|k_access|k_acc_keys|k_walker" -c 8 \
  -o gpurun_out/full_$W python profiles/run_one.py --workload $W --repeat 1 > gpurun_out/ncu_f_$W.log 2>&1
for f in gpurun_out/ncu_l_$W.log gpurun_out/ncu_f_$W.log; do tail -n 1 $f; done
