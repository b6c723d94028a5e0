set -x
timeout 1200 python -m pytest tests/test_gpu_small.py -q -x > gpurun_out/small_tests.log 2>&1
tail -30 gpurun_out/small_tests.log
python tools/small_batch_latency.py > gpurun_out/small_latency.txt 2>&1
cat gpurun_out/small_latency.txt
timeout 1800 python -m pytest tests/test_ref_suite.py -m gpu -q -s -k "acceptance or update or render" > gpurun_out/ref_suite_acc.log 2>&1
grep -E "criterion|passed|failed" gpurun_out/ref_suite_acc.log | tail -30
