# parity + per-phase trace + bench (no cpu) in one call
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/perf_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 4 gpurun_out/perf_pytest.log
timeout 300 python tools/phase_trace.py --batches 20 > gpurun_out/perf_phase.txt 2>&1; tail -n 9 gpurun_out/perf_phase.txt
timeout 600 python bench.py --no-cpu > gpurun_out/perf_bench.json 2>gpurun_out/perf_bench.err
python -c "import json; d=json.load(open('gpurun_out/perf_bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], d['batch_ms'], d['phase_ms']['median_ms'])"
