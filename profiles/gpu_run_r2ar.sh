#!/bin/bash
# interpolated stamp lookups in long hard-event lists
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -2
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/br_c4.json 2> gpurun_out/br_c4.err
tail -n 1 gpurun_out/br_c4.err
python -c "
import json; d=json.load(open('gpurun_out/br_c4.json')); print('c4', d['ms_per_step'], d['e2e']['value'], d['kernel_ms_eager'])"
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/br_c5.json 2> gpurun_out/br_c5.err
python -c "
import json; d=json.load(open('gpurun_out/br_c5.json')); print('c5', d['ms_per_step'], d['e2e']['value'])"
