#!/bin/bash
# A/B timing of alternative builds in one GPU session: bash tools/ab.sh lib1.so lib2.so ...
for rep in 1 2; do
for lib in "$@"; do
  PB_LIB_PATH=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 32768 ${AB_ARGS} | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],4), round(d['ms_per_step'],2))"
done
done
