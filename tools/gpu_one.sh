# run one pytest selection on the GPU: bash tools/gpu_one.sh <pytest args...>
timeout 1200 python -m pytest -q -x "$@" > gpurun_out/one_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 25 gpurun_out/one_pytest.log
