#!/bin/bash
# Run on the GPU box: plain bench then one ncu --set full capture of the decode kernel.
# usage: bash tools/prof.sh TAG [bench args...]   (env PB_* passes through)
tag=$1; shift
args="--batch 4096 --steps 1 --warmup 3 --no-cpu-baseline $*"
python bench.py $args > gpurun_out/${tag}_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_decode -s 3 -c 1 -o gpurun_out/${tag} python bench.py $args > gpurun_out/${tag}_ncu.log 2>&1
echo "prof rc=$?"
