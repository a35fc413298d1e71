#!/bin/bash
# A/B of alternative library builds over several configs in one GPU session:
#   bash tools/ab_cfg.sh "cfg1 cfg2" lib1.so lib2.so ...
cfgs=$1; shift
for rep in 1 2; do
for c in $cfgs; do
for lib in "$@"; do
  PB_LIB_PATH=$lib timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch 32768 ${AB_ARGS} 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$(basename $lib)', round(d['value'],4))" || echo "$c $lib FAILED"
done; done; done
