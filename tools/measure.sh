#!/bin/bash
# Full measurement pass on the GPU box (round evidence):
#   bench line (default config), ncu launch list of the same command, one
#   ncu --set full capture of the decode kernel, per-op cycles (profiling build).
# usage: bash tools/measure.sh TAG
tag=${1:-m}
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_launch.log 2>&1
bash tools/prof.sh ${tag}_full
python tools/op_cycles.py c3_L32 > gpurun_out/${tag}_op_cycles.txt 2>&1
echo done
