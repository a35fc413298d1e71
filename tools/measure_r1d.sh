#!/bin/bash
# Round-end measurement refresh (run on the GPU box): GPU tests, default bench
# line, reference arm, launch list, all configs, per-op cycles.
tag=${1:-r1d}
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -1 gpurun_out/${tag}_tests.log
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -c 400 gpurun_out/${tag}_bench.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_launch.log 2>&1
bash tools/bench_all.sh > gpurun_out/${tag}_all.txt 2>&1; cat gpurun_out/${tag}_all.txt
python tools/op_cycles.py c3_L32 > gpurun_out/${tag}_op_cycles.txt 2>&1
echo done
