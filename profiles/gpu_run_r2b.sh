set -x
timeout 1800 python tests/golden/make_full_digests.py --out gpurun_out/full_digests.json 2>&1 | tail -40
cp gpurun_out/full_digests.json tests/golden/full_digests.json
timeout 900 python -m pytest tests/test_gpu_fullscale.py -x -q 2>&1 | tail -15
