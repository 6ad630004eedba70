timeout 900 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_exchange.py -x -q --tb=short 2>&1 | tail -5
GW_XS_DEBUG=1 GW_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_x2.json 2> gpurun_out/bench_x2.err; grep "gw xs\|Error" gpurun_out/bench_x2.err | head; cut -c1-1800 gpurun_out/bench_x2.json
GW_BUCKET=2 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; python -c "
import json; d=json.load(open('gpurun_out/bench_s.json')); print(d['ms_per_step'], d['gpu_launches'], d['kernel_ms_eager'])"
