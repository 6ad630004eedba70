timeout 1800 python -m pytest tests -x -q -m gpu --tb=short --deselect tests/test_gpu_exchange.py 2>&1 | tail -15
for v in 0 1; do GW_BUCKET=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p$v.json 2> gpurun_out/bench_p$v.err; python -c "
import json; d=json.load(open('gpurun_out/bench_p$v.json')); print('bucket=$v', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['kernel_ms_eager'])"; done
