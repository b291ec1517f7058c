#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/dyn_tests.log 2>&1
for lib in base dyn; do
for rep in 1 2; do
FL_LIB=tools/_ab/lib_$lib.so timeout 120 python tools/attn_bench.py 144 256 16 700 >> gpurun_out/ab5_att_$lib.log 2>&1
FL_LIB=tools/_ab/lib_$lib.so timeout 120 python tools/attn_bench.py 64 96 64 1055 >> gpurun_out/ab5_att_$lib.log 2>&1
FL_LIB=tools/_ab/lib_$lib.so timeout 120 python tools/attn_bench.py 144 256 16 3000 >> gpurun_out/ab5_att_$lib.log 2>&1
done
FL_LIB=tools/_ab/lib_$lib.so timeout 300 python tools/prof_step.py --config c3 --rows 128 --pre 300 --iters 20 >> gpurun_out/ab5_step_$lib.log 2>&1
done
