timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_small.py tests/test_gpu_delta.py tests/test_gpu_streams.py -q -x 2>&1 | tail -3
for m in 0 1 2 0 1 2; do
  LOD_COUNT_STAGED=$m timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/ab_$m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$m.json')); print('mode $m', d['value'], d['e2e']['value'], d['batch_ms'], d['phase_ms']['median_ms']['count'])"
done
python tools/sorted_vs_shuffled.py 2>&1 | tail -2
