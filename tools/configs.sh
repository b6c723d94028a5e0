# bench every config shape (device + e2e), no CPU baseline / rows
for c in uniform skew mesh; do
  timeout 900 python bench.py --config $c --no-cpu --no-rows --steps ${1:-95} > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  python -c "import json; d=json.load(open('gpurun_out/cfg_$c.json')); print('$c', d['value'], d['e2e']['value'], d['batch_ms'], d['config']['final_nodes'])" || tail -n 5 gpurun_out/cfg_$c.err
done
