#!/bin/bash
# closing bench lines of C4 / C3 / C2 on the final build
set -u
mkdir -p gpurun_out
for w in c4 c3 c2; do
  st=5; [ $w = c3 ] && st=3; [ $w = c2 ] && st=20
  timeout 1200 python bench.py --workload $w --steps $st --warmup 3 > gpurun_out/r2i_bench_$w.json 2> gpurun_out/r2i_bench_$w.err
  tail -n 1 gpurun_out/r2i_bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/r2i_bench_$w.json')); print('$w', d['ms_per_step'], d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['cpu_baseline']['value'], d['python_reference']['value'])"
done
