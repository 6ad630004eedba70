set -x
timeout 600 python -m pytest tests/test_gpu_bucket.py -x -q 2>&1 | tail -30
timeout 2000 python tests/golden/make_full_digests.py --out gpurun_out/full_digests.json 2>&1 | tail -20
cp gpurun_out/full_digests.json tests/golden/full_digests.json
timeout 900 python -m pytest tests/test_gpu_fullscale.py -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_bk.json 2> gpurun_out/bench_c5_bk.err; tail -5 gpurun_out/bench_c5_bk.err; cat gpurun_out/bench_c5_bk.json
