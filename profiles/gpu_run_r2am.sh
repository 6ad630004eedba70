#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bp_decode" -c 1 \
  -o gpurun_out/r2_full_bp3 python profiles/run_delta.py c5 bp > gpurun_out/ncu_fbp.log 2>&1; tail -n 1 gpurun_out/ncu_fbp.log
