#!/bin/bash
# ncu --set full capture of the specialised lane kernel (c3 L=32, 16384 frames) after a plain run
tag=${1:-jit}; shift
args="--batch 16384 --steps 1 --warmup 3 --no-cpu-baseline --no-latency $*"
python bench.py $args > gpurun_out/${tag}_plain.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pb_lane_jit -s 3 -c 1 -o gpurun_out/${tag} python bench.py $args > gpurun_out/${tag}_ncu.log 2>&1
echo "prof rc=$?"
