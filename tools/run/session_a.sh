set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/small_batch_latency.py > gpurun_out/small_latency.txt 2>&1
timeout 2400 python -m pytest tests/test_ref_suite.py -m gpu -q -x -s -k "not acceptance" > gpurun_out/ref_suite.log 2>&1
timeout 1800 python -m pytest tests/test_ref_suite.py -m gpu -q -s -k "acceptance" > gpurun_out/ref_suite_acc.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --ignore=tests/test_ref_suite.py > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
