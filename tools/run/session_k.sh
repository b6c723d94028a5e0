LOD_COUNT_STAGED=1 bash tools/ncu_kernel.sh "k_count" 10 kcount_staged_r02
