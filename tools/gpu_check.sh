# quick GPU check: parity tests (+ optional bench).  gpurun -- bash tools/gpu_check.sh [bench]
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/chk_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 15 gpurun_out/chk_pytest.log
if [ "$1" = "bench" ]; then
timeout 600 python bench.py --no-cpu > gpurun_out/chk_bench.json 2>gpurun_out/chk_bench.err; head -c 400 gpurun_out/chk_bench.json
fi
