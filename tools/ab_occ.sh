#!/bin/bash
# Occupancy sweep: library variant x frames per SM x first global beta slot.
L=paper_1505_01466_b200/_lib
run() { lab=$1; lib=$2; cfg=$3; shift 3
  env PB_LIB_PATH=$lib "$@" timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --batch 32768 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['plan']; print('$cfg $lab', round(d['value'],4), p['frames_per_sm'], p['smem_per_frame'], p['alpha_global_from_stage'], p['global_scratch_per_frame'])" || echo "$cfg $lab FAILED"
}
for c in ${CFGS:-c3_L32 c5_L16}; do
run t512_f16_b7 $L/var_t512.so $c PB_FRAMES_PER_SM=16 PB_BETA_GLOBAL_FROM=7
run t512_f16_b6 $L/var_t512.so $c PB_FRAMES_PER_SM=16 PB_BETA_GLOBAL_FROM=6
run t512_f16_b5 $L/var_t512.so $c PB_FRAMES_PER_SM=16 PB_BETA_GLOBAL_FROM=5
run t640_f20_b7 $L/var_t640.so $c PB_FRAMES_PER_SM=20 PB_BETA_GLOBAL_FROM=7
run t640_f20_b6 $L/var_t640.so $c PB_FRAMES_PER_SM=20 PB_BETA_GLOBAL_FROM=6
run t640_f20_b5 $L/var_t640.so $c PB_FRAMES_PER_SM=20 PB_BETA_GLOBAL_FROM=5
run t768_f24_b6 $L/var_t768.so $c PB_FRAMES_PER_SM=24 PB_BETA_GLOBAL_FROM=6
run t768_f24_b5 $L/var_t768.so $c PB_FRAMES_PER_SM=24 PB_BETA_GLOBAL_FROM=5
done
