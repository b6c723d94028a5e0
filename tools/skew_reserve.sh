# skew bench vs pool reserve size
for r in 6144 16384 24576; do
  LOD_DEBUG=1 LOD_POOL_RESERVE_MIB=$r timeout 900 python bench.py --config skew --no-cpu --no-rows > gpurun_out/skr.json 2> gpurun_out/skr.err
  python -c "import json; d=json.load(open('gpurun_out/skr.json')); print('[reserve $r]', d['value'], d['e2e']['value'], d['batch_ms'])"
  grep "pool reserve" gpurun_out/skr.err
done
