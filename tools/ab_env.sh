#!/bin/bash
# Env / variant sweep on one box:  CFGS="..." bash tools/ab_env.sh
L=paper_1505_01466_b200/_lib
run() { lab=$1; lib=$2; cfg=$3; shift 3
  env PB_LIB_PATH=$lib "$@" timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --batch 32768 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['plan']; print('$cfg $lab', round(d['value'],4), p['frames_per_sm'], p['smem_per_frame'], p['alpha_global_from_stage'])" || echo "$cfg $lab FAILED"
}
for c in ${CFGS:-c3_L32}; do
run base $L/libpolar_b200.so $c
run sync15 $L/libpolar_b200.so $c PB_SYNC_MASK=15
run sync63 $L/libpolar_b200.so $c PB_SYNC_MASK=63
run nosync $L/libpolar_b200.so $c PB_SYNC_MASK=-1
run fps14 $L/libpolar_b200.so $c PB_FRAMES_PER_SM=14
run uq42 $L/var_uq42.so $c
run uq44 $L/var_uq44.so $c
run base $L/libpolar_b200.so $c
done
