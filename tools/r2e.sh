python tools/op_cycles.py c3_L32 > gpurun_out/r2e_op_cycles.txt 2>&1; cat gpurun_out/r2e_op_cycles.txt
