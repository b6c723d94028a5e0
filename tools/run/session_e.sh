timeout 1200 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_small.py -q 2>&1 | tail -4
python tools/sorted_vs_shuffled.py 2>&1 | tail -4
