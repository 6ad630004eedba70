#!/bin/bash
# k_hard_append_w: four windows' loads per warp iteration
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -2
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bq_c4.json 2> gpurun_out/bq_c4.err
tail -n 1 gpurun_out/bq_c4.err
python -c "
import json; d=json.load(open('gpurun_out/bq_c4.json')); print('c4', d['ms_per_step'], d['e2e']['value'], d['kernel_ms_eager'])"
