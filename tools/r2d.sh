bash tools/ab_lane.sh "PB_LANE=1" "PB_LIB_PATH=paper_1505_01466_b200/_lib/libpolar_b200_v2rt.so"
python tools/op_cycles.py c3_L32 > gpurun_out/r2d_op_cycles.txt 2>&1; head -30 gpurun_out/r2d_op_cycles.txt
