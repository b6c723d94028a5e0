# where the big skew batch (batch 11: 5.9M spill, 7.45M new voxels) spends its time
LOD_DEBUG=2 timeout 300 python tools/stream_trace.py --config skew --batches 14 > gpurun_out/skew_trace.txt 2> gpurun_out/skew_trace.err
grep "batch" gpurun_out/skew_trace.txt | tail -n 5
grep -v "^\[lod\] batch" gpurun_out/skew_trace.err | tail -n 40
