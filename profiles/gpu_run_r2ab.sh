#!/bin/bash
# k_access register double buffering; graph-mode launch list (k_ingest) and full-set captures
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullscale.py -x -q --tb=short 2>&1 | tail -3
for I in 1 0; do
  GW_INGEST=$I timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bb_c5_$I.json 2> gpurun_out/bb_c5_$I.err
  tail -n 1 gpurun_out/bb_c5_$I.err
  python -c "
import json; d=json.load(open('gpurun_out/bb_c5_$I.json')); print('c5 ingest=$I', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_c5_graph.csv \
    python profiles/run_one.py --workload c5 --repeat 3 --graph > gpurun_out/ncu_lg.log 2>&1; tail -n 1 gpurun_out/ncu_lg.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ingest|k_access" -c 2 \
  -o gpurun_out/r2_full_c5_ab python profiles/run_one.py --workload c5 --repeat 2 --graph > gpurun_out/ncu_fab.log 2>&1; tail -n 1 gpurun_out/ncu_fab.log
