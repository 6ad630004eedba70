timeout 900 python -m pytest tests/test_gpu_packed.py -x -q --tb=short 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; tail -3 gpurun_out/r2_bench_c5.err; python -c "
import json; d=json.load(open('gpurun_out/r2_bench_c5.json')); print(d['ms_per_step'], json.dumps(d['e2e']), d['roofline']['kernel'], d['roofline']['frac'], d.get('python_reference'), d['cpu_baseline'])"
