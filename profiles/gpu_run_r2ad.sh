#!/bin/bash
# lock walker: read-only pre-check in w_fused_join (no object for joins that change nothing)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullscale.py tests/test_gpu_integration.py -x -q --tb=short 2>&1 | tail -2
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bd_c3.json 2> gpurun_out/bd_c3.err
tail -n 1 gpurun_out/bd_c3.err
python -c "
import json; d=json.load(open('gpurun_out/bd_c3.json')); print('c3', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
GW_PROF_WALKER=1 timeout 600 python profiles/run_one.py --workload c3 --repeat 1 2>&1 | grep -i "walker\|C3" | tail -3
