# per-kernel warm-cache durations of one steady-state batch (serialised by ncu, no cache flush)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv \
  --log-file gpurun_out/warm_launches.csv python tools/profile_run.py --warmup ${1:-11} --profiled 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/warm_launches.csv
