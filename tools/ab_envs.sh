# A/B environment settings on the default bench (same build): bash tools/ab_envs.sh "" "VAR=1" "VAR=2" ...
for rep in 1 2; do
  for e in "$@"; do
    env $e timeout 600 python bench.py --no-cpu --no-rows > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('[$e]', d['value'], d['e2e']['value'], d['batch_ms']['p50'])"
  done
done
