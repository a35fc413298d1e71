#!/bin/bash
# Round-2 re-entry check (GPU box): GPU tests, default bench, ncu --set full of the lane kernel at 16384 frames, per-op cycles.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_tests.log 2>&1; tail -2 gpurun_out/r2h_tests.log
python bench.py --no-cpu-baseline > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; tail -c 400 gpurun_out/r2h_bench.json
args="--batch 16384 --steps 1 --warmup 3 --no-cpu-baseline --no-latency"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lane -s 3 -c 1 -o gpurun_out/r2h_lane python bench.py $args > gpurun_out/r2h_ncu.log 2>&1
echo "ncu rc=$?"
python tools/op_cycles.py c3_L32 > gpurun_out/r2h_op_cycles.txt 2>&1; head -30 gpurun_out/r2h_op_cycles.txt
