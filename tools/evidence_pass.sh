#!/bin/bash
# usage (one GPU): gpurun -- bash tools/evidence_pass.sh   -> $OUT (default gpurun_out/final)
# tests, smoke, compute-sanitizer on attention, launch list + ncu (profile_round.sh),
# algorithmic bytes, CUPTI step trace, bench lines for C3 / C4 / C2 / the reference arm
# round-end evidence pass (one GPU)
O=${OUT:-gpurun_out/final}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_kernels.py -q -k "attention or attn or shuffle" > $O/sanitize_memcheck_attention.log 2>&1; echo "rc=$?" >> $O/sanitize_memcheck_attention.log
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_kernels.py -q -k "attention or attn" > $O/sanitize_racecheck_attention.log 2>&1; echo "rc=$?" >> $O/sanitize_racecheck_attention.log
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_kernels.py -q -k "attention or attn" > $O/sanitize_synccheck_attention.log 2>&1; echo "rc=$?" >> $O/sanitize_synccheck_attention.log
OUT=$O CFG=c3 ROWS=144 PRE=350 timeout 1500 bash tools/profile_round.sh > $O/profile.log 2>&1
timeout 600 python tools/prof_step.py --config c3 --rows 144 --pre 350 --iters 2 --profile --dump $O/alg_c3.json > $O/alg_c3.log 2>&1
timeout 600 python tools/trace_step.py --config c3 --rows 128 --iters 5 --json $O/trace_c3.json > $O/trace_c3.log 2>&1
timeout 900 python bench.py > $O/bench_c3.log 2>&1
timeout 900 python bench.py --config c4 --steps 2 > $O/bench_c4.log 2>&1
timeout 900 python bench.py --config c2 --steps 3 > $O/bench_c2.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1
echo done > $O/done
