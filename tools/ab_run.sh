# A/B every abtmp/v*.so on the default bench, interleaved, N reps
cat abtmp/variants.txt 2>/dev/null
for rep in $(seq ${1:-2}); do
  for L in abtmp/v*.so; do
    LOD_B200_LIB=$L timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$L', d['value'], d['e2e']['value'], d['batch_ms']['p50'])"
  done
done
