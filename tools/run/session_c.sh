set -x
free -g | head -2; nproc
timeout 2400 python -m pytest tests -m gpu -q -x --ignore=tests/test_ref_suite.py > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
timeout 1800 python -m pytest tests/test_ref_suite.py -m gpu -q -s > gpurun_out/ref_suite_all.log 2>&1
grep -E "criterion|passed|failed|FAILED" gpurun_out/ref_suite_all.log | tail -40
