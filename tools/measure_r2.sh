#!/bin/bash
# Round-2 measurement refresh (run on the GPU box): GPU tests, default bench
# line, reference arm, launch list, all configs, per-op cycles (16 frames per
# SM and one frame alone), full-volume parity, torchrun (world size 1) bench,
# one ncu --set full capture of the decode kernel at the bench batch.
tag=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -1 gpurun_out/${tag}_tests.log
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -c 300 gpurun_out/${tag}_bench.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-latency > gpurun_out/${tag}_launch.log 2>&1
bash tools/bench_all.sh > gpurun_out/${tag}_all.txt 2>&1; cat gpurun_out/${tag}_all.txt
python tools/op_cycles.py c3_L32 > gpurun_out/${tag}_op_cycles.txt 2>&1
OPC_FRAMES=1 python tools/op_cycles.py c3_L32 > gpurun_out/${tag}_op_cycles_1frame.txt 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_torchrun.json 2> gpurun_out/${tag}_torchrun.err
tail -c 200 gpurun_out/${tag}_torchrun.json
args="--steps 1 --warmup 3 --no-cpu-baseline --no-latency"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pb_lane_jit -s 3 -c 1 -o gpurun_out/${tag}_ncu_c3_L32 \
    python bench.py $args > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
python tools/parity_full.py gpu --out gpurun_out/${tag}_parity_full.json > gpurun_out/${tag}_parity.log 2>&1; tail -3 gpurun_out/${tag}_parity.log
echo done
