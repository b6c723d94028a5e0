timeout 1200 python -m pytest tests/test_gpu_small.py -q -x 2>&1 | tail -40
