#!/bin/bash
# correctness across warps-per-frame settings, then bench per setting (dev helper)
for w in 1 2 4 8; do
  echo "== PB_WARPS=$w"; PB_WARPS=$w timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
done
