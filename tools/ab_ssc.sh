L=paper_1505_01466_b200/_lib
run() { lab=$1; lib=$2; cfg=$3; shift 3
  env PB_LIB_PATH=$lib "$@" timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --batch 65536 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['plan']['ssc']; print('$cfg $lab', round(d['value'],4), p)" || echo "$cfg $lab FAILED"
}
for c in c3_L1 c3_L32_adaptive c5_L16_adaptive; do
run ssc512 $L/var_ssc512.so $c
run d1024 $L/libpolar_b200.so $c
run d1024_f24 $L/libpolar_b200.so $c PB_SSC_FPC=24
run d1024_f16smem $L/libpolar_b200.so $c PB_SSC_FPC=16 PB_SSC_CH_GLOBAL=0
done
