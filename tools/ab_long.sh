# A/B every abtmp/v*.so on a long terrain stream (N batches)
for L in abtmp/v*.so; do
  LOD_B200_LIB=$L timeout 1200 python tools/long_stream.py --batches ${1:-400} --arena-gib 32 --window 200 2>&1 | tail -n 3 | sed "s|^|$L |"
done
