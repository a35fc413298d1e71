timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; python -c "import json; d=json.load(open('gpurun_out/r2g_bench.json')); print(d['value'], d['e2e'], d['latency'], d['roofline']['frac'])" || tail -5 gpurun_out/r2g_bench.err
python bench.py --config c4_int8_L32 --steps 5 --no-cpu-baseline > gpurun_out/r2g_c4.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/r2g_c4.json')); print(d['value'], d['e2e'], d['latency'])"
python tools/time_python_reference.py --config c3_L32 --min-seconds 60 --out gpurun_out/r2g_pyref_c3_L32.json
