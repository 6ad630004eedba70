#!/bin/bash
# balanced digit widths in the big sort (k_rs_up / k_rs_down_tma templated on RB <= 8)
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/be_c5.json 2> gpurun_out/be_c5.err
tail -n 1 gpurun_out/be_c5.err
python -c "
import json; d=json.load(open('gpurun_out/be_c5.json')); print('c5', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/be_c4.json 2> gpurun_out/be_c4.err
tail -n 1 gpurun_out/be_c4.err
python -c "
import json; d=json.load(open('gpurun_out/be_c4.json')); print('c4', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_c5_graph2.csv \
    python profiles/run_one.py --workload c5 --repeat 3 --graph > gpurun_out/ncu_lg2.log 2>&1; tail -n 1 gpurun_out/ncu_lg2.log
