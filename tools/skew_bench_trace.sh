# host timeline of every insert in the skew bench; print the slow ones with their growth lines
LOD_DEBUG=2 timeout 600 python bench.py --config skew --no-cpu --no-rows --steps ${1:-95} > gpurun_out/skb.json 2> gpurun_out/skb.err
python -c "import json; d=json.load(open('gpurun_out/skb.json')); print(d['value'], d['batch_ms'])"
python - <<'PY'
import re
lines = open("gpurun_out/skb.err").read().splitlines()
pend = []
nb = 0
for l in lines:
    if "timeline" in l:
        nb += 1
        last = int(re.findall(r"=(\d+)", l)[-1])
        if last > 3000:
            print("call", nb, "host us", last)
            for p in pend[-12:]:
                print("   ", p)
            print("   ", l[:400])
        pend = []
    elif "batch n=" not in l:
        pend.append(l)
print("calls", nb)
PY
