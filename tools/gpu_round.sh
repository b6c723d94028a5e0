#!/bin/bash
# One GPU-box session: parity tests, smoke, bench, ncu launch list + full capture.
#   gpurun --timeout 1500 -- bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
tail -3 $OUT/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/${TAG}_smoke.log
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"; tail -c 1500 $OUT/${TAG}_bench.json
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $OUT/${TAG}_launches.csv python tools/profile_run.py --warmup 11 --profiled 1 > /dev/null 2>&1
python tools/launch_summary.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launch_summary.txt 2>&1; head -12 $OUT/${TAG}_launch_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o $OUT/${TAG}_full -f python tools/profile_run.py --warmup 11 --profiled 1 > $OUT/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
