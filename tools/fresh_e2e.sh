# first bench process on a fresh box: e2e check (run as the first command of a gpurun call)
timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/fresh.json 2>gpurun_out/fresh.err
python -c "import json; d=json.load(open('gpurun_out/fresh.json')); print('[fresh]', d['value'], d['e2e']['value'], d['batch_ms']['p50'])"
