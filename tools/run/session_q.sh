( time timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_20.json 2> gpurun_out/bench_20.err ) 2> gpurun_out/bench_20.time
tail -3 gpurun_out/bench_20.err; cat gpurun_out/bench_20.time
timeout 1500 python bench.py > gpurun_out/bench_95.json 2> gpurun_out/bench_95.err; tail -3 gpurun_out/bench_95.err
python -c "
import json
for f in ('bench_20', 'bench_95'):
    d=json.load(open('gpurun_out/'+f+'.json'))
    print(f, d['value'], d['e2e']['value'], d['batch_ms'])
    print(json.dumps(d['rows']['disk_ingest']))
    print(json.dumps(d['rows']['small_batches']))
"
