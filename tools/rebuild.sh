#!/bin/bash
# rebuild the CUDA library in-tree (from any cwd); prints errors only
cd "$(dirname "$0")/.." && python -m paper_2310_03567_b200.build "$@" 2>&1 | grep -iE "error|warning" | head -20
ls -la --time-style=+%T paper_2310_03567_b200/_lodb200.so | awk '{print $6, $7}'
