#!/bin/bash
# Per-shape ncu metrics of the C3 projection GEMMs (one GPU; cold L2, serialised launches).
#   OUT=gpurun_out/x bash tools/gemm_shape_ncu.sh  -> $OUT/gemm_shape_<part>_<M>.csv
# then: python tools/gemm_shape_ncu.py $OUT > profiles/<round>_gemm_per_shape_ncu.csv
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
MET=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for part in in out lm; do
  for M in ${MS:-8 64 128 144 192 256 320}; do
    # the eager warm-up pass of step_gemm_bench launches the part once per layer: skip 4, take 4
    ONLY=$part timeout 300 ncu --metrics $MET --clock-control none -k regex:k_gemm_sk -s 4 -c 4 --csv \
      --log-file $OUT/gemm_shape_${part}_${M}.csv python tools/step_gemm_bench.py $M > $OUT/gemm_shape_${part}_${M}.log 2>&1
  done
done
