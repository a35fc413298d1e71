mkdir -p gpurun_out
python -c "
import paper_1505_01466_b200 as pb, json
spec=pb.CodeSpec.from_design_ebn0(2048,1691,pb.CRC32,4.0); sch=pb.build_schedule(spec)
d=pb.ListDecoder(sch,32); print(d.plan)
"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2b_tests.log; tail -30 gpurun_out/r2b_tests.log
for c in c3_L32 c4_int8_L32; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_$c.json 2>gpurun_out/r2b_$c.err; python -c "import json; d=json.load(open('gpurun_out/r2b_$c.json')); print('$c', d['value'], d['roofline']['frac'])" || tail -5 gpurun_out/r2b_$c.err; done
