timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_small.py -q -x 2>&1 | tail -2
for i in 1 2; do
  timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/ab_x.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_x.json')); print('now', d['value'], d['e2e']['value'], d['batch_ms']['p50'], d['phase_ms']['median_ms'])"
done
python tools/sorted_vs_shuffled.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_ref_suite.py -m gpu -q -s -k "acceptance" > gpurun_out/ref_suite_o.log 2>&1
grep -E "criterion|passed|failed|FAILED" gpurun_out/ref_suite_o.log | tail -20
