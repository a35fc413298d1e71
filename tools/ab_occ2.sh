L=paper_1505_01466_b200/_lib
run() { lab=$1; lib=$2; cfg=$3; shift 3
  env PB_LIB_PATH=$lib "$@" timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --batch 32768 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['plan']; print('$cfg $lab', round(d['value'],4), p['frames_per_sm'], p['smem_per_frame'], p['alpha_global_from_stage'], p['global_scratch_per_frame'])" || echo "$cfg $lab FAILED"
}
for c in c3_L32 c5_L16 c4_int8_L32; do
run base $L/libpolar_b200.so $c
run t384_f12 $L/var_t384.so $c PB_FRAMES_PER_SM=12
run t448_f14 $L/var_t448.so $c PB_FRAMES_PER_SM=14
run persist64 $L/libpolar_b200.so $c PB_L2_PERSIST=64
run persist100 $L/libpolar_b200.so $c PB_L2_PERSIST=100
run base $L/libpolar_b200.so $c
done
