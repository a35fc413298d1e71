#!/bin/bash
# A/B of decoder options on the GPU box: bash tools/ab.sh CONFIG "opt=val,opt=val" ... ("-" = defaults)
cfg=$1; shift
for setting in "$@"; do
  args=""
  if [ "$setting" != "-" ]; then for kv in ${setting//,/ }; do args="$args --opt $kv"; done; fi
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-latency $args > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$cfg', '$setting', round(d['value'],3), 'e2e', round(d['e2e']['value'],3))" || tail -3 gpurun_out/ab.err
done
