LOD_DEBUG=2 timeout 300 python tools/stream_trace.py --config terrain --batches 30 > gpurun_out/timeline.txt 2>&1
grep timeline gpurun_out/timeline.txt | tail -n 12
