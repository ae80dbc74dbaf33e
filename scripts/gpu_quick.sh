#!/usr/bin/env bash
# Quick GPU check: gemm tests, C3 phase timing (and optional env overrides), bench.
#   gpurun -- 'bash scripts/gpu_quick.sh <tag> [pytest-args]'
set -u
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
shift || true
if [ $# -gt 0 ]; then
  ( timeout 900 python -m pytest "$@" -x -q 2>&1 | tail -15 ) > $OUT/pytest.log
  tail -3 $OUT/pytest.log
fi
timeout 300 python scripts/profile_update.py --N 4096 --epochs 3 --updates 3 > $OUT/c3.log 2>&1
tail -1 $OUT/c3.log
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
  echo "bench rc=$?"; cat $OUT/bench.json; tail -3 $OUT/bench.err
fi
