timeout 2000 python -m pytest tests -x -q -m gpu --tb=short 2>&1 | tail -15
GW_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_x2.json 2> gpurun_out/bench_x2.err; tail -3 gpurun_out/bench_x2.err; cut -c1-1500 gpurun_out/bench_x2.json
