L=paper_1505_01466_b200/_lib
run() { lab=$1; lib=$2; cfg=$3; shift 3
  env PB_LIB_PATH=$lib "$@" timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --batch 32768 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['plan']; print('$cfg $lab', round(d['value'],4), p['frames_per_sm'], p['warps_per_frame'], p['smem_per_frame'], p['alpha_global_from_stage'], p['global_scratch_per_frame'])" || echo "$cfg $lab FAILED"
}
for c in c3_L32 c5_L16; do
run w1 $L/var_head.so $c
run w2f8 $L/var_head.so $c PB_WARPS=2 PB_FRAMES_PER_SM=8
run w2f8b8 $L/var_head.so $c PB_WARPS=2 PB_FRAMES_PER_SM=8 PB_BETA_GLOBAL_FROM=9
run w4f4 $L/var_head.so $c PB_WARPS=4 PB_FRAMES_PER_SM=4
run w4f4b11 $L/var_head.so $c PB_WARPS=4 PB_FRAMES_PER_SM=4 PB_BETA_GLOBAL_FROM=13
done
