#!/bin/bash
# Frames per SM for the small-L shapes (launch bound variants): bash tools/ab_small_l.sh
L=paper_1505_01466_b200/_lib
run() { lab=$1; lib=$2; cfg=$3; shift 3
  env PB_LIB_PATH=$lib "$@" timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --batch 32768 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['plan']; print('$cfg $lab', round(d['value'],4), p['frames_per_sm'], p['smem_per_frame'], p['alpha_global_from_stage'])" || echo "$cfg $lab FAILED"
}
for c in ${CFGS:-c1_L4 c3_L2 c3_L8 c2_L8}; do
run base $L/libpolar_b200.so $c
run t768_f24 $L/var_t768.so $c PB_FRAMES_PER_SM=24
run t1024_f32 $L/var_t1024.so $c PB_FRAMES_PER_SM=32
run t1024_f24 $L/var_t1024.so $c PB_FRAMES_PER_SM=24
done
