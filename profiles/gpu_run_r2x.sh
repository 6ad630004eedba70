#!/bin/bash
# lazy access stamps (k_access<.., true>, no k_acc_aux): GPU suite, C5/C2 bench lazy vs aux, ncu of k_access
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -5
for L in 1 0; do
  GW_ACC_LAZY=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bx_c5_$L.json 2> gpurun_out/bx_c5_$L.err
  python -c "
import json; d=json.load(open('gpurun_out/bx_c5_$L.json')); print('c5 lazy=$L', d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
  GW_ACC_LAZY=$L timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bx_c2_$L.json 2> gpurun_out/bx_c2_$L.err
  python -c "
import json; d=json.load(open('gpurun_out/bx_c2_$L.json')); print('c2 lazy=$L', d['ms_per_step'], d['e2e']['value'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_access" -c 1 \
  -o gpurun_out/r2_full_c5_klazy python profiles/run_one.py --workload c5 --repeat 1 > gpurun_out/ncu_fl.log 2>&1; tail -n 1 gpurun_out/ncu_fl.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_c5_lazy.csv \
    python profiles/run_one.py --workload c5 --repeat 1 > gpurun_out/ncu_ll.log 2>&1; tail -n 1 gpurun_out/ncu_ll.log
