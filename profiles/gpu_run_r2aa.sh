#!/bin/bash
# k_ingest (fused prep / keys / first digit counts / hard events), single-thread fast path, delta-upload race fix
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
for I in 1 0; do
  GW_INGEST=$I timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ba_c5_$I.json 2> gpurun_out/ba_c5_$I.err
  tail -n 1 gpurun_out/ba_c5_$I.err
  python -c "
import json; d=json.load(open('gpurun_out/ba_c5_$I.json')); print('c5 ingest=$I', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
done
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ba_c2.json 2> gpurun_out/ba_c2.err
python -c "
import json; d=json.load(open('gpurun_out/ba_c2.json')); print('c2', d['ms_per_step'], d['e2e']['value'])"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_c5_aa.csv \
    python profiles/run_one.py --workload c5 --repeat 1 > gpurun_out/ncu_laa.log 2>&1; tail -n 1 gpurun_out/ncu_laa.log
