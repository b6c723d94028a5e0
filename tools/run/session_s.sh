timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_delta.py -q -x 2>&1 | tail -2
for m in 0 64 0 64; do
  LOD_RESOLVE_LIST_MAX_MB=$m timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/ab_$m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$m.json')); p=d['phase_ms']['median_ms']; print('list<=${m}MB', d['value'], d['e2e']['value'], d['batch_ms']['p50'], p['resolve'], p['backlog'])"
done
