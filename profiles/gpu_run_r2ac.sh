#!/bin/bash
# k_ingest with batched loads
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullscale.py -x -q --tb=short 2>&1 | tail -2
for I in 1 0; do
  GW_INGEST=$I timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bc_c5_$I.json 2> gpurun_out/bc_c5_$I.err
  tail -n 1 gpurun_out/bc_c5_$I.err
  python -c "
import json; d=json.load(open('gpurun_out/bc_c5_$I.json')); print('c5 ingest=$I', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ingest" -c 1 \
  -o gpurun_out/r2_full_c5_ingest python profiles/run_one.py --workload c5 --repeat 2 --graph > gpurun_out/ncu_fi.log 2>&1; tail -n 1 gpurun_out/ncu_fi.log
