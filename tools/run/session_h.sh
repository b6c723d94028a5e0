python tools/c9_probe.py 2>&1 | tail -6
python tools/sorted_vs_shuffled.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_small.py tests/test_gpu_fuzz.py tests/test_gpu_multiproc.py tests/test_ingest.py -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_ref_suite.py -m gpu -q -s -k "octree or acceptance" > gpurun_out/ref_suite_h.log 2>&1
grep -E "criterion|passed|failed|FAILED" gpurun_out/ref_suite_h.log | tail -24
bash tools/ncu_kernel.sh k_count 10 kcount_r02 ; ls -la gpurun_out/kcount_r02*
