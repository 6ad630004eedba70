set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
free -g | head -2; nproc
python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_fullscale.py 2>&1 | tail -5
timeout 1500 python tests/golden/make_full_digests.py --out gpurun_out/full_digests.json 2>&1 | tail -40
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err; cat gpurun_out/bench_c5.json
