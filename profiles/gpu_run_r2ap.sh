#!/bin/bash
# C4: lazy stamp lookups vs the per-event aux pass
set -u
mkdir -p gpurun_out
for L in 1 0; do
GW_ACC_LAZY=$L timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bp_c4_$L.json 2> gpurun_out/bp_c4_$L.err
tail -n 1 gpurun_out/bp_c4_$L.err
python -c "
import json; d=json.load(open('gpurun_out/bp_c4_$L.json')); print('c4 lazy=$L', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['kernel_ms_eager'] if 'kernel_ms_eager' in d else '')"
done
