#!/bin/bash
mkdir -p gpurun_out
for lib in base cw8; do
for rep in 1 2; do
FL_LIB=tools/_ab/lib_$lib.so timeout 120 python tools/attn_bench.py 144 256 16 700 >> gpurun_out/ab4_att_$lib.log 2>&1
FL_LIB=tools/_ab/lib_$lib.so timeout 120 python tools/attn_bench.py 64 96 64 1055 >> gpurun_out/ab4_att_$lib.log 2>&1
FL_LIB=tools/_ab/lib_$lib.so timeout 120 python tools/attn_bench.py 144 256 16 300 >> gpurun_out/ab4_att_$lib.log 2>&1
done
FL_LIB=tools/_ab/lib_$lib.so timeout 300 python tools/prof_step.py --config c3 --rows 128 --pre 300 --iters 20 >> gpurun_out/ab4_step_$lib.log 2>&1
done
