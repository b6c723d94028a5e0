timeout 1500 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_peer.py tests/test_gpu_route.py tests/test_gpu_multiproc.py tests/test_ingest.py -q -x 2>&1 | tail -15
timeout 2400 python -m pytest tests/test_gpu_scale.py -q -s -x > gpurun_out/scale.log 2>&1
grep -E "config|passed|failed|Error|assert" gpurun_out/scale.log | tail -20
