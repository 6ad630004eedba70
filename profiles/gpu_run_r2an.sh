#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_packed.py -x -q --tb=short -k bitpacked 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_bp_decode" --log-file gpurun_out/r2_launches_c5_bp2.csv \
  python profiles/run_delta.py c5 bp > gpurun_out/ncu_lbp2.log 2>&1; tail -n 1 gpurun_out/ncu_lbp2.log
