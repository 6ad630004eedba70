#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --tb=short 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/by_c5.json 2> gpurun_out/by_c5.err
tail -n 2 gpurun_out/by_c5.err
python -c "
import json; d=json.load(open('gpurun_out/by_c5.json')); print('c5', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
