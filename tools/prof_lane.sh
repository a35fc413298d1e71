# ncu full capture of the lane kernel (c3 L=32, 4096 frames) + plain run
tag=${1:-lane}; shift
args="--batch 4096 --steps 1 --warmup 3 --no-cpu-baseline $*"
python bench.py $args > gpurun_out/${tag}_plain.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_lane -s 3 -c 1 -o gpurun_out/${tag} python bench.py $args > gpurun_out/${tag}_ncu.log 2>&1
echo "prof rc=$?"
