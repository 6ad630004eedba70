timeout 1500 python -m pytest tests -x -q -m gpu --tb=short 2>&1 | tail -25
