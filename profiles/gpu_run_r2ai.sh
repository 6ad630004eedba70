#!/bin/bash
# k_access occupancy experiment (__launch_bounds__(256, 5) for the lazy variant)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullscale.py -x -q --tb=short 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bi_c5.json 2> gpurun_out/bi_c5.err
tail -n 1 gpurun_out/bi_c5.err
python -c "
import json; d=json.load(open('gpurun_out/bi_c5.json')); print('c5', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_access" -c 1 --csv python profiles/run_one.py --workload c5 --repeat 1 2>/dev/null | grep k_access | tail -2
