L=paper_1505_01466_b200/_lib
run() { # label lib envs...
  lab=$1; lib=$2; shift 2
  env PB_LIB_PATH=$lib "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 32768 ${AB_ARGS} 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['plan']; print('$lab', round(d['value'],4), p['frames_per_sm'], p['smem_per_frame'], p['alpha_global_from_stage'], p['warps_per_frame'])" || echo "$lab FAILED"
}
for rep in 1 2; do
run base $L/libpolar_b200.so
run t384_w1_f12 $L/var_t384.so PB_FRAMES_PER_SM=12
run t512_w1_f16 $L/var_t512.so PB_FRAMES_PER_SM=16
run t512_w2_f8 $L/var_t512.so PB_WARPS=2
run t384_w2_f6 $L/var_t384.so PB_WARPS=2 PB_FRAMES_PER_SM=6
run t512_w1_f8 $L/var_t512.so
done
