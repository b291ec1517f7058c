#!/bin/bash
# One-GPU profiling pass for the round's evidence (run under gpurun).
#   launch list (every kernel of steady-state fused iterations, cold cache)
#   + ncu --set full of the top kernels (attention, projection GEMM, shuffle)
set -u
OUT=${OUT:-gpurun_out}
CFG=${CFG:-c3}
ROWS=${ROWS:-256}
mkdir -p $OUT
# launch list: skip admission passes + warm-up iterations, then ~2 iterations
# (prof_step brackets its steady-state decode loop with cudaProfilerStart/Stop)
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c ${COUNT:-240} --csv --log-file $OUT/launches_${CFG}.csv \
    python tools/prof_step.py --config $CFG --rows $ROWS --pre ${PRE:-350} --iters 2 > $OUT/launches_${CFG}.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_attn_tma -c 1 \
    -o $OUT/attn_${CFG} python tools/prof_step.py --config $CFG --rows $ROWS --pre ${PRE:-350} --iters 2 > $OUT/attn_${CFG}.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gemm_sk -c 5 \
    -o $OUT/gemm_${CFG} python tools/prof_step.py --config $CFG --rows $ROWS --pre ${PRE:-350} --iters 2 > $OUT/gemm_${CFG}.log 2>&1
ncu --set full --clock-control none -k regex:k_shuffle -s 3 -c 1 \
    -o $OUT/shuffle python tools/shuffle_bench.py 512 2 > $OUT/shuffle.log 2>&1
echo profile done
