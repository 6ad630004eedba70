#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullscale.py -x -q --tb=short 2>&1 | tail -2
for W in 1 0; do
GW_ACC_WORK=$W timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bk_c5_$W.json 2> gpurun_out/bk_c5_$W.err
tail -n 1 gpurun_out/bk_c5_$W.err
python -c "
import json; d=json.load(open('gpurun_out/bk_c5_$W.json')); print('c5 work=$W', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_access" -c 2 --csv python profiles/run_one.py --workload c5 --repeat 1 2>/dev/null | grep k_access | tail -2
