# A/B of lane-kernel runtime knobs on c3 L=32 (and int8): value Gbit/s per setting
cfg=${CFG:-c3_L32}
for setting in "$@"; do
  env $setting timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$cfg', '$setting', round(d['value'],3), 'e2e', round(d['e2e']['value'],3))" || tail -3 gpurun_out/ab.err
done
