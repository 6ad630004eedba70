#!/bin/bash
# Round-2 closing run: GPU suite, the C5 bench line (default command), the reference arm
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -3
timeout 1200 python bench.py > gpurun_out/r2j_bench_c5.json 2> gpurun_out/r2j_bench_c5.err
tail -n 1 gpurun_out/r2j_bench_c5.err
python -c "
import json; d=json.load(open('gpurun_out/r2j_bench_c5.json')); print('c5', d['ms_per_step'], d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['cpu_baseline']['value'], d['python_reference']['value'], d['clocks'], d['gpu_launches'], d['steps'], d['warmup'])"
timeout 900 python bench.py --impl reference > gpurun_out/r2j_bench_ref_c5.json 2> gpurun_out/r2j_bench_ref_c5.err
python -c "
import json; d=json.load(open('gpurun_out/r2j_bench_ref_c5.json')); print('ref', d['value'], d['cpu_baseline'])"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
