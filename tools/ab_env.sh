# A/B of an environment switch on the default bench: bash tools/ab_env.sh VAR=VALUE
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/ab_a.json 2>/dev/null
  env "$1" timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/ab_b.json 2>/dev/null
  python -c "
import json; a=json.load(open('gpurun_out/ab_a.json')); b=json.load(open('gpurun_out/ab_b.json'))
print('default', a['value'], a['e2e']['value'], '| $1', b['value'], b['e2e']['value'])"
done
