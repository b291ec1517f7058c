#!/bin/bash
mkdir -p gpurun_out
timeout 200 python tools/step_gemm_bench.py 8 64 144 256 > gpurun_out/elect.log 2>&1
ONLY=in GEMM_DBG=1 timeout 200 python tools/step_gemm_bench.py 8 144 >> gpurun_out/elect.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_merged.py -x -q > gpurun_out/elect_tests.log 2>&1
