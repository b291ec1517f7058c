#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "argmax or lm_head" > gpurun_out/e8b_tests.log 2>&1
for o in out lm; do ONLY=$o timeout 200 python tools/step_gemm_bench.py 8 64 144 256 >> gpurun_out/e8b.log 2>&1; done
for o in out lm; do ONLY=$o FL_LIB=tools/_ab/lib_pre8.so timeout 200 python tools/step_gemm_bench.py 8 64 144 256 >> gpurun_out/e8b.log 2>&1; done
