#!/bin/bash
# k_access: positions needing the full check flagged in the blocked scan pass, checked from a list
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bg_c5.json 2> gpurun_out/bg_c5.err
tail -n 1 gpurun_out/bg_c5.err
python -c "
import json; d=json.load(open('gpurun_out/bg_c5.json')); print('c5', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bg_c4.json 2> gpurun_out/bg_c4.err
python -c "
import json; d=json.load(open('gpurun_out/bg_c4.json')); print('c4', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bg_c2.json 2> gpurun_out/bg_c2.err
python -c "
import json; d=json.load(open('gpurun_out/bg_c2.json')); print('c2', d['ms_per_step'], d['e2e']['value'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_access" -c 1 \
  -o gpurun_out/r2_full_c5_klist python profiles/run_one.py --workload c5 --repeat 1 > gpurun_out/ncu_fl2.log 2>&1; tail -n 1 gpurun_out/ncu_fl2.log
