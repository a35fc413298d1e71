#!/bin/bash
# A/B of the recomputed stage n-2 (PB_VIRT2) over configs: CFGS="..." bash tools/ab_virt2.sh
for c in ${CFGS:-c3_L32 c4_int8_L32 c5_L16 c3_L8 c2_L8 c1_L4 c3_L2}; do
  for v in 0 1; do
    PB_VIRT2=$v timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch 32768 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['plan']; print('$c virt2=$v', round(d['value'],4), p.get('virt2'), p['frames_per_sm'], p['alpha_global_from_stage'])" || echo "$c virt2=$v FAILED"
  done
done
