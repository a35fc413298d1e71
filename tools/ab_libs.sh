#!/bin/bash
# A/B of library builds on one box, interleaved (label=path pairs):
#   CFGS="c3_L32 ..." bash tools/ab_libs.sh head=paper_1505_01466_b200/_lib/var_head.so new=paper_1505_01466_b200/_lib/libpolar_b200.so
for c in ${CFGS:-c3_L32 c4_int8_L32 c5_L16 c3_L8}; do
  for rep in 1 2; do
    for lv in "$@"; do
      lab=${lv%%=*}; lib=${lv#*=}
      env PB_LIB_PATH=$lib ${AB_ENV} timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch ${AB_BATCH:-32768} 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $lab', round(d['value'],4))" || echo "$c $lab FAILED"
    done
  done
done
