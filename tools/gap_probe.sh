# device time of batch 19 vs the sum of its kernels (warm ncu, serialised)
timeout 300 python tools/stream_trace.py --config terrain --batches 20 2>&1 | grep "batch  19"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv \
  --log-file gpurun_out/gap_launches.csv python tools/profile_run.py --warmup 19 --profiled 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/gap_launches.csv | tail -n 1
