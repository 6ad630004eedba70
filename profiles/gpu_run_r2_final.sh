#!/bin/bash
# Round-2 final measurements: GPU suite, bench lines of C5 (default) / C4 / C3 / C2 with the
# CPU baselines, the reference arm on C5, graph-mode launch lists and full-set captures.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -3
for w in c5 c4 c3 c2; do
  st=5; [ $w = c3 ] && st=3; [ $w = c2 ] && st=20
  timeout 1200 python bench.py --workload $w --steps $st --warmup 3 > gpurun_out/r2g_bench_$w.json 2> gpurun_out/r2g_bench_$w.err
  tail -n 1 gpurun_out/r2g_bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/r2g_bench_$w.json')); print('$w', d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['cpu_baseline']['value'], d.get('python_reference'), d['clocks'])"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2g_bench_ref_c5.json 2> gpurun_out/r2g_bench_ref_c5.err
tail -c 400 gpurun_out/r2g_bench_ref_c5.json
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for w in c5 c4; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2g_launches_$w.csv \
    python profiles/run_one.py --workload $w --repeat 3 --graph > gpurun_out/ncu_r2g_$w.log 2>&1; tail -n 1 gpurun_out/ncu_r2g_$w.log
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_rs_down_tma|k_access|k_ingest" -c 4 \
  -o gpurun_out/r2g_full_c5 python profiles/run_one.py --workload c5 --repeat 2 --graph > gpurun_out/ncu_r2g_full.log 2>&1; tail -n 1 gpurun_out/ncu_r2g_full.log
