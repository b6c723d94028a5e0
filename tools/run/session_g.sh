timeout 2400 python -m pytest tests -m gpu -q --ignore=tests/test_ref_suite.py --ignore=tests/test_gpu_scale.py > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
timeout 1500 python -m pytest tests/test_ref_suite.py -m gpu -q -s > gpurun_out/ref_suite_all.log 2>&1
grep -E "criterion|passed|failed|FAILED" gpurun_out/ref_suite_all.log | tail -30
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_20.json 2> gpurun_out/bench_20.err
tail -c 3000 gpurun_out/bench_20.json; tail -5 gpurun_out/bench_20.err
timeout 3000 python -m pytest tests/test_gpu_scale.py -q -s -x > gpurun_out/scale.log 2>&1
tail -30 gpurun_out/scale.log
