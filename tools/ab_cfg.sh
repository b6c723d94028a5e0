# A/B abtmp/v0.so vs abtmp/v1.so on a config: bash tools/ab_cfg.sh <config> [reps]
for rep in $(seq ${2:-2}); do
  for L in abtmp/v0.so abtmp/v1.so; do
    LOD_B200_LIB=$L timeout 600 python bench.py --config $1 --no-cpu --no-rows > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$1 $L', d['value'], d['e2e']['value'], d['batch_ms'])"
  done
done
