python tools/kineto_gaps.py --warm 20 --batches 4 > gpurun_out/timeline_r02.txt 2>&1; tail -80 gpurun_out/timeline_r02.txt
