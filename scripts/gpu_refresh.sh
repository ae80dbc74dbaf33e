#!/usr/bin/env bash
# round-2 refresh: GPU tests, smoke, bench + reference arm, C3 profile (launch list, trace, ncu)
set -u
T=${1:-r02s}
OUT=gpurun_out/$T
mkdir -p $OUT
( timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 ) > $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 ) > $OUT/smoke.log
tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; head -c 300 $OUT/bench.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2>>$OUT/bench.err
bash scripts/c3_profile.sh $T > $OUT/c3_profile.out 2>&1
head -12 $OUT/c3_launches_summary.txt
# summaries on the box; the big reports stay behind (gpurun merges <= 64 MiB back)
for r in $OUT/prof_c3_gru_step_gemm0 $OUT/prof_c3_gru_step_gemm1 $OUT/prof_c3_tc_gemm; do
  [ -f $r.ncu-rep ] && python scripts/ncu_summary.py $r.ncu-rep "$(basename $r) ($T)" > $r.md 2>/dev/null
done
rm -f $OUT/prof_c3_tc_gemm.ncu-rep $OUT/c3_launches.csv
ls -la $OUT | head -30
