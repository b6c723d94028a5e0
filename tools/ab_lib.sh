# A/B two builds on the same box: bash tools/ab_lib.sh <libA.so> <libB.so> [reps]
for rep in $(seq ${3:-3}); do
  for L in "$1" "$2"; do
    LOD_B200_LIB=$L timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$L', d['value'], d['e2e']['value'], d['batch_ms']['p50'])"
  done
done
