timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cn in 1 2 4; do FL_SK_VERBOSE=1 FL_SK_CN=$cn timeout 600 python tools/layer_gemm_bench.py 320 128 8 2>&1 | sort | uniq | sed "s/^/cn=$cn /"; done
