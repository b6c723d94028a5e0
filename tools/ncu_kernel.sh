# full ncu capture of selected kernels of one batch: bash tools/ncu_kernel.sh <regex> <warmup> <tag>
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:$1" \
  -o gpurun_out/$3 -f python tools/profile_run.py --warmup $2 --profiled 1 > gpurun_out/$3.log 2>&1; echo "ncu rc=$?"
