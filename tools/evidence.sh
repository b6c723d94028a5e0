# round-end bench evidence: default terrain line (with CPU baseline + rows), every other config's line
timeout 900 python bench.py > gpurun_out/ev_terrain.json 2> gpurun_out/ev_terrain.err
python -c "import json; d=json.load(open('gpurun_out/ev_terrain.json')); print('terrain', d['value'], d['e2e']['value'], d['batch_ms'])" || tail -n 5 gpurun_out/ev_terrain.err
for c in uniform skew mesh; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/ev_$c.json 2> gpurun_out/ev_$c.err
  python -c "import json; d=json.load(open('gpurun_out/ev_$c.json')); print('$c', d['value'], d['e2e']['value'], d['batch_ms'], d['config']['final_nodes'])" || tail -n 5 gpurun_out/ev_$c.err
done
