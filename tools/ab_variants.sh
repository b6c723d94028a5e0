# build the default and variants (nvcc -D flags) into abtmp/, then A/B them on the box
#   bash tools/ab_variants.sh "-DFOO=1" "-DBAR=2" ...   (run here, then gpurun tools/ab_run.sh)
mkdir -p abtmp; rm -f abtmp/*.so abtmp/variants.txt
python -m paper_2310_03567_b200.build --force > /dev/null && cp paper_2310_03567_b200/_lodb200.so abtmp/v0.so
i=1
for v in "$@"; do
  LOD_NVCC_EXTRA="$v" python -m paper_2310_03567_b200.build --force > /dev/null && cp paper_2310_03567_b200/_lodb200.so abtmp/v$i.so
  echo "v$i: $v" >> abtmp/variants.txt
  i=$((i+1))
done
python -m paper_2310_03567_b200.build --force > /dev/null
