#!/bin/bash
# ncu --set full of the C5 access-pass kernels (k_access, k_acc_aux, k_acc_tilemax, k_rs_up)
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_access|k_acc_aux|k_acc_tilemax|k_rs_up" -c 4 \
  -o gpurun_out/r2_full_c5_access python profiles/run_one.py --workload c5 --repeat 1 > gpurun_out/ncu_fa.log 2>&1; tail -n 3 gpurun_out/ncu_fa.log
