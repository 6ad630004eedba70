#!/bin/bash
# Round-2 profiling (run under gpurun from the repo root; outputs in gpurun_out/):
# launch lists (gpu__time_duration + DRAM bytes per launch) of one eager C5 / C4
# analysis on the default (LSD) pass and on the bucketed pass, the delta-decode
# kernels of an end-to-end C5 analysis, and ncu --set full of the top kernels.
set -u
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for W in c5 c4; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_$W.csv \
    python profiles/run_one.py --workload $W --repeat 1 > gpurun_out/ncu_l_$W.log 2>&1; tail -n 1 gpurun_out/ncu_l_$W.log
  GW_BUCKET=2 timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_${W}_bucket.csv \
    python profiles/run_one.py --workload $W --repeat 1 > gpurun_out/ncu_lb_$W.log 2>&1; tail -n 1 gpurun_out/ncu_lb_$W.log
done
timeout 900 ncu --metrics $M --clock-control none --csv -k regex:"k_delta_decode|k_widen" --log-file gpurun_out/r2_launches_c5_delta.csv \
  python profiles/run_delta.py c5 > gpurun_out/ncu_ld.log 2>&1; tail -n 1 gpurun_out/ncu_ld.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rs_down_tma|k_access|k_acc_keys" -c 3 \
  -o gpurun_out/r2_full_c5 python profiles/run_one.py --workload c5 --repeat 1 > gpurun_out/ncu_f.log 2>&1; tail -n 1 gpurun_out/ncu_f.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_delta_decode" -c 2 \
  -o gpurun_out/r2_full_delta python profiles/run_delta.py c5 > gpurun_out/ncu_fd.log 2>&1; tail -n 1 gpurun_out/ncu_fd.log
