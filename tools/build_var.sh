#!/bin/bash
# Build an experiment variant of the library with extra nvcc defines and a
# subset of the shapes:  bash tools/build_var.sh NAME "-DPB_MAXT=512 ..." [shape,shape]
name=$1; defs=$2; shapes=${3:-f32_w1_p32_chg,f32_w1_p16_chg,f32_w1_p8_chg,i8_w1_p32,f32_w1_p4,f32_w1_p2,f32_w1_p1,i8_w1_p1,f32_w1_p1_chg}
PB_NVCC_DEFS="$defs" PB_SHAPES="$shapes" PB_LIB_OUT=$PWD/paper_1505_01466_b200/_lib/var_$name.so \
  python -c "from paper_1505_01466_b200 import _native; _native.build()"
