#!/bin/bash
# k_access carry by decoupled look-back (no k_acc_tilemax), tiles taken in order
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
for L in 1 0; do
GW_ACC_LOOKBACK=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bo_c5_$L.json 2> gpurun_out/bo_c5_$L.err
tail -n 1 gpurun_out/bo_c5_$L.err
python -c "
import json; d=json.load(open('gpurun_out/bo_c5_$L.json')); print('c5 lb=$L', d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'])"
done
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bo_c2.json 2> gpurun_out/bo_c2.err
python -c "
import json; d=json.load(open('gpurun_out/bo_c2.json')); print('c2', d['ms_per_step'], d['e2e']['value'])"
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bo_c4.json 2> gpurun_out/bo_c4.err
python -c "
import json; d=json.load(open('gpurun_out/bo_c4.json')); print('c4', d['ms_per_step'], d['e2e']['value'])"
