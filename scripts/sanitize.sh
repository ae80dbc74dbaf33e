#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize.py
#   gpurun -- 'bash scripts/sanitize.sh <tag>'
set -u
OUT=gpurun_out/${1:-san}
mkdir -p $OUT
timeout 300 python scripts/sanitize.py > $OUT/plain.log 2>&1; echo "plain rc=$?"; cat $OUT/plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize.py \
    > $OUT/$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 $OUT/$tool.log
done
