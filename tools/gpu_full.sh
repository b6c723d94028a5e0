# round evidence: parity tests, smoke, default bench (with CPU baseline), warm launch list, ncu full capture
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log; tail -n 3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'cpu', d['cpu_baseline'], d['roofline'])"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>&1; tail -c 300 gpurun_out/${TAG}_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/profile_run.py --warmup 11 --profiled 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_summary.txt; head -n 8 gpurun_out/${TAG}_launch_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o gpurun_out/${TAG}_full -f python tools/profile_run.py --warmup 11 --profiled 1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
