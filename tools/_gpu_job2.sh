#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_merged.py tests/test_gpu_fullshape.py -x -q > gpurun_out/gfast_tests.log 2>&1
ONLY=in timeout 200 python tools/step_gemm_bench.py 64 144 256 > gpurun_out/gfast.log 2>&1
timeout 200 python tools/step_gemm_bench.py 8 64 144 256 >> gpurun_out/gfast.log 2>&1
