python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
( time timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1 ) 2> gpurun_out/pytest_time.txt
tail -8 gpurun_out/pytest_gpu_full.log; cat gpurun_out/pytest_time.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_20.json 2> gpurun_out/bench_20.err; tail -3 gpurun_out/bench_20.err
timeout 1200 python bench.py > gpurun_out/bench_95.json 2> gpurun_out/bench_95.err; tail -3 gpurun_out/bench_95.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2>&1
python -c "
import json
for f in ('bench_20','bench_95','bench_ref'):
    d=json.load(open('gpurun_out/'+f+'.json'))
    print(f, d['value'], d.get('e2e',{}).get('value'), d.get('batch_ms'), (d.get('roofline') or {}).get('traffic'))
"
