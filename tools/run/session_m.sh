timeout 1200 python -m pytest tests/test_gpu_scale.py -q -s -k "past_2_24" 2>&1 | tail -5
bash tools/ncu_traffic.sh terrain 5 20
bash tools/ncu_traffic.sh terrain 5 95
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/render_r02 -f python tools/render_profile.py --warmup 25 > gpurun_out/render_r02.log 2>&1; echo "render ncu rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python tools/profile_run.py --warmup 11 --profiled 1 > /dev/null 2>&1; echo "launches rc=$?"
