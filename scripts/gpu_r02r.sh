#!/usr/bin/env bash
# round-2 refresh: bench + reference arm, C3 trace / launch list / ncu of the step kernels
set -u
T=${1:-r02r}
OUT=gpurun_out/$T
mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; head -c 400 $OUT/bench.json; echo
bash scripts/c3_profile.sh $T > $OUT/c3_profile.out 2>&1
tail -30 $OUT/c3_profile.out
