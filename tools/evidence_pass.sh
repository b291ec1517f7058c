#!/bin/bash
# usage (one GPU): gpurun -- bash tools/evidence_pass.sh   -> $OUT (default gpurun_out/final)
# tests, smoke, launch list + ncu (profile_round.sh),
# algorithmic bytes, CUPTI step trace, bench lines for C3 / C4 / C2 / the reference arm
# round-end evidence pass (one GPU)
O=${OUT:-gpurun_out/final}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
# compute-sanitizer runs: profiles/r02c_sanitize_*, profiles/r02n_sanitize_* (the tool is closed on this pool since)
OUT=$O CFG=c3 ROWS=144 PRE=350 timeout 1500 bash tools/profile_round.sh > $O/profile.log 2>&1
timeout 600 python tools/prof_step.py --config c3 --rows 144 --pre 350 --iters 2 --profile --dump $O/alg_c3.json > $O/alg_c3.log 2>&1
timeout 600 python tools/trace_step.py --config c3 --rows 128 --iters 5 --json $O/trace_c3.json > $O/trace_c3.log 2>&1
timeout 900 python bench.py > $O/bench_c3.log 2>&1
timeout 900 python bench.py --config c4 --steps 2 > $O/bench_c4.log 2>&1
timeout 900 python bench.py --config c2 --steps 3 > $O/bench_c2.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1
echo done > $O/done
