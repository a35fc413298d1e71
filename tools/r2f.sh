timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/ab_lane.sh "PB_LANE=1"
CFG=c4_int8_L32 bash tools/ab_lane.sh "PB_LANE=1"
