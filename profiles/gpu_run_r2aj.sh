#!/bin/bash
# k_access flagged positions to a worklist drained by k_access_work
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
for W in 1 0; do
GW_ACC_WORK=$W timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bj_c5_$W.json 2> gpurun_out/bj_c5_$W.err
tail -n 1 gpurun_out/bj_c5_$W.err
python -c "
import json; d=json.load(open('gpurun_out/bj_c5_$W.json')); print('c5 work=$W', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
done
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bj_c4.json 2> gpurun_out/bj_c4.err
python -c "
import json; d=json.load(open('gpurun_out/bj_c4.json')); print('c4', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_c5_graph4.csv \
    python profiles/run_one.py --workload c5 --repeat 3 --graph > gpurun_out/ncu_lg3.log 2>&1; tail -n 1 gpurun_out/ncu_lg3.log
