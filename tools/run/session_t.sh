timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_streams.py tests/test_gpu_multiproc.py -q -x 2>&1 | tail -2
for i in 1 2; do
  timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/ab_x.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_x.json')); p=d['phase_ms']['median_ms']; print('now', d['value'], d['e2e']['value'], d['batch_ms']['p50'])"
done
python tools/kineto_gaps.py --warm 20 --batches 4 2>&1 | tail -3
