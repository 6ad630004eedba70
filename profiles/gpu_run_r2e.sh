timeout 600 python -m pytest tests/test_gpu_bucket.py -x -q --tb=short 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; tail -3 gpurun_out/bench_e.err; python -c "
import json; d=json.load(open('gpurun_out/bench_e.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_ms_eager'])"
