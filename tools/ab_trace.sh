# per-batch device ms of the default stream for every abtmp/v*.so, side by side
for L in abtmp/v*.so; do
  LOD_B200_LIB=$L timeout 600 python tools/stream_trace.py --batches ${1:-60} 2>&1 | grep "^rep" | awk '{print $6}' > gpurun_out/$(basename $L).ms
done
paste gpurun_out/v*.so.ms | awk '{d=$2-$1; printf "%3d %s %s %+.3f\n", NR-1, $1, $2, d}' | sort -k4 -g -r | head -n 12
