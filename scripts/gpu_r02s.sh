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
