#!/bin/bash
# bit-packed host trace (GWSOA v4): device decoder parity, bench legs, decoder launch times
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_packed.py -x -q --tb=short 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bl_c5.json 2> gpurun_out/bl_c5.err
tail -n 2 gpurun_out/bl_c5.err
python -c "
import json; d=json.load(open('gpurun_out/bl_c5.json')); e=d['e2e']; print('c5', d['ms_per_step'], e['value'], e['ms_per_step'], e['h2d_bytes_per_step'], 'delta', e['delta']['value'], e['delta']['ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_bp_decode" --log-file gpurun_out/r2_launches_c5_bp.csv \
  python profiles/run_delta.py c5 bp > gpurun_out/ncu_lbp.log 2>&1; tail -n 1 gpurun_out/ncu_lbp.log
