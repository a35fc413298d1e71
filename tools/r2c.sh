timeout 600 python -m pytest tests -m gpu -x -q -k "lane or L32 or 32 or oracle or parity_volume or golden or dropin" 2>&1 | tail -3
bash tools/ab_lane.sh "PB_LANE=1"
CFG=c4_int8_L32 bash tools/ab_lane.sh "PB_LANE=1"
python tools/op_cycles.py c3_L32 > gpurun_out/r2c_op_cycles.txt 2>&1; head -40 gpurun_out/r2c_op_cycles.txt
