#!/bin/bash
# One short bench line per config (device-resident value, e2e, roofline fraction).
# usage: bash tools/bench_all.sh [configs...]
cfgs=${@:-"c1_L4 c2_L8 c3_L1 c3_L2 c3_L8 c3_L32 c4_int8_L32 c5_L16 c3_L32_adaptive c2_L8_adaptive c4_int8_L32_adaptive c5_L16_adaptive"}
for c in $cfgs; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ba_$c.json 2>gpurun_out/ba_$c.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ba_$c.json')); print('$c', round(d['value'],3), 'e2e', round(d['e2e']['value'],3), 'frac', round(d['roofline']['frac'],4), 'inv', d.get('list_invoked_frac'))" || tail -3 gpurun_out/ba_$c.err
done
