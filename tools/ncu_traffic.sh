# DRAM bytes per launch of every update kernel over bench.py's timed batch
# range (config stream batches W .. W+K-1, the same seeds and tree), for the
# bench line's roofline.traffic:   bash tools/ncu_traffic.sh <config> <W> <K>
# -> gpurun_out/traffic_<config>_<W>_<K>.csv; then
#    python tools/ncu_traffic.py gpurun_out/traffic_*.csv  (merges into profiles/ncu_traffic.json)
CFG=${1:-terrain}; W=${2:-5}; K=${3:-20}
GEN=$(python -c "import bench; print(bench.CONFIGS['$CFG'][0])")
timeout 1500 ncu --profile-from-start off --clock-control none --cache-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file gpurun_out/traffic_${CFG}_${W}_${K}.csv \
  python tools/profile_run.py --config $GEN --warmup $W --profiled $K > gpurun_out/traffic_${CFG}_${W}_${K}.log 2>&1
echo "ncu rc=$?"
