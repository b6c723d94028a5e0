LOD_DEBUG=1 timeout 600 python tools/stream_trace.py --config terrain --batches 100 --repeat 2 > gpurun_out/trace_terrain.txt 2>&1
for c in uniform skew mesh; do timeout 300 python tools/stream_trace.py --config $c --batches 20 > gpurun_out/trace_$c.txt 2>&1; done
tail -3 gpurun_out/trace_*.txt
