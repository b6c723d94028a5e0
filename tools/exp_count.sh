# k_count experiments: claim statistics (LOD_EXP_COUNT) and the no-claim timing bound (LOD_EXP_NOCLAIM)
LOD_NVCC_EXTRA="-DLOD_EXP_COUNT" python -m paper_2310_03567_b200.build --force > /dev/null 2>&1
timeout 300 python tools/phase_trace.py --batches 20 2>&1 | grep "claims=" | tail -n 5
LOD_NVCC_EXTRA="-DLOD_EXP_NOCLAIM" python -m paper_2310_03567_b200.build --force > /dev/null 2>&1
timeout 300 python tools/phase_trace.py --batches 20 2>&1 | tail -n 4
python -m paper_2310_03567_b200.build --force > /dev/null 2>&1
timeout 300 python tools/phase_trace.py --batches 20 2>&1 | tail -n 4
