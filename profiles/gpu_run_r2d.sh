set -x
timeout 600 python -m pytest tests/test_gpu_bucket.py -x -q --tb=short 2>&1 | tail -40
timeout 600 python -m pytest tests/test_gpu_packed.py -x -q --tb=short 2>&1 | tail -20
timeout 2000 python tests/golden/make_full_digests.py --out gpurun_out/full_digests.json 2>&1 | tail -20
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bk_down|k_bk_check|k_bk_up" -c 4 -o gpurun_out/ncu/r2_c5_bk python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bk.log 2>&1; tail -5 gpurun_out/ncu_bk.log
