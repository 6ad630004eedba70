timeout 1200 python -m pytest tests/test_gpu_exchange.py -x -q --tb=short 2>&1 | tail -30
timeout 1500 python -m pytest tests -x -q -m gpu --tb=short --deselect tests/test_gpu_exchange.py 2>&1 | tail -15
