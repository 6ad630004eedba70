#!/bin/bash
# one-round stamp lookups for short hard-event lists; sentinel-free location keys (few non-access events)
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
for S in 0 1; do
GW_SENTINEL=$S timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bh_c5_$S.json 2> gpurun_out/bh_c5_$S.err
tail -n 1 gpurun_out/bh_c5_$S.err
python -c "
import json; d=json.load(open('gpurun_out/bh_c5_$S.json')); print('c5 sentinel=$S', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
done
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bh_c2.json 2> gpurun_out/bh_c2.err
python -c "
import json; d=json.load(open('gpurun_out/bh_c2.json')); print('c2', d['ms_per_step'], d['e2e']['value'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_access" -c 1 \
  -o gpurun_out/r2_full_c5_kstamp python profiles/run_one.py --workload c5 --repeat 1 > gpurun_out/ncu_fl3.log 2>&1; tail -n 1 gpurun_out/ncu_fl3.log
