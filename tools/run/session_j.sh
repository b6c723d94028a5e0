timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -2
for m in 0 1 0 1; do
  LOD_COUNT_STAGED=$m timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/ab_$m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$m.json')); print('mode $m', d['value'], d['e2e']['value'], d['batch_ms']['p50'], d['phase_ms']['median_ms']['count'])"
done
