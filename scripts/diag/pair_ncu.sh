#!/usr/bin/env bash
# Why does the CTA-pair step kernel fail under ncu?  (diagnostics, one gpurun call)
set -u
OUT=gpurun_out/${1:-pair}
mkdir -p $OUT
P="python scripts/profile_update.py --N 1024 --epochs 1 --updates 1"
timeout 300 $P > $OUT/plain.log 2>&1; echo "plain rc=$?"; tail -2 $OUT/plain.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gru_step_gemm2 -c 1 $P > $OUT/ncu_default.log 2>&1; echo "ncu default rc=$?"; grep -E "ERROR|duration" $OUT/ncu_default.log | head -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:gru_step_gemm2 -c 1 $P > $OUT/ncu_nocache.log 2>&1; echo "ncu nocache rc=$?"; grep -E "ERROR|duration" $OUT/ncu_nocache.log | head -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --replay-mode application -k regex:gru_step_gemm2 -c 1 $P > $OUT/ncu_app.log 2>&1; echo "ncu app rc=$?"; grep -E "ERROR|duration" $OUT/ncu_app.log | head -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_gemm2 -c 1 $P > $OUT/ncu_gemm2.log 2>&1; echo "ncu gemm2 rc=$?"; grep -E "ERROR|duration" $OUT/ncu_gemm2.log | head -3
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 $P > $OUT/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 $OUT/memcheck.log
