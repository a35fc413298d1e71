mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r2a_tests.log 2>&1; tail -1 gpurun_out/r2a_tests.log
python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; tail -c 600 gpurun_out/r2a_bench.json
python tools/op_cycles.py c3_L32 > gpurun_out/r2a_op_cycles.txt 2>&1; head -40 gpurun_out/r2a_op_cycles.txt
