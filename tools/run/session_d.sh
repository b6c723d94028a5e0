python tools/run/diag_fuzz.py 40 2>&1 | tail -30
echo ---- pipeline only
LOD_NO_SMALL=1 python tools/run/diag_fuzz.py 40 2>&1 | tail -8
timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q 2>&1 | tail -8
