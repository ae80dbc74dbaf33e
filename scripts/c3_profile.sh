#!/usr/bin/env bash
# C3 (configs[2]) evidence in one gpurun call: plain phase timing, the per-step
# recurrence trace, the ncu launch list of one update, ncu --set full of the
# top GEMMs and both step-kernel directions.
#   gpurun -- 'bash scripts/c3_profile.sh <tag>'
set -u
OUT=gpurun_out/${1:-c3}
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
P="python scripts/profile_update.py --N 4096 --epochs 3"
timeout 600 $P --updates 2 > $OUT/c3_plain.log 2>&1
tail -1 $OUT/c3_plain.log
rm -f /tmp/c3_trace.txt
VER_REC_TRACE=/tmp/c3_trace.txt timeout 600 $P --updates 1 > $OUT/c3_trace.log 2>&1
cp /tmp/c3_trace.txt $OUT/c3_trace.txt 2>/dev/null
python scripts/step_trace.py $OUT/c3_trace.txt > $OUT/c3_step_trace.txt 2>&1
python scripts/rec_trace.py $OUT/c3_trace.txt > $OUT/c3_rec_trace.txt 2>&1
cat $OUT/c3_step_trace.txt | head -40
[ "${NCU:-1}" = "1" ] || exit 0
export VER_PROFILING=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/c3_launches.csv $P --updates 2 > $OUT/c3_launches.log 2>&1
echo "launch list rc=$?"
python scripts/launches.py $OUT/c3_launches.csv 0.5 40 > $OUT/c3_launches_summary.txt 2>&1
cat $OUT/c3_launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 40 -c 6 \
  -o $OUT/prof_c3_tc_gemm $P --updates 1 > $OUT/prof_c3_tc_gemm.log 2>&1
for d in 0 1; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:gru_step_gemm2?_kernel<.{0,5}$d(, .{0,8})?>" -s 2 -c 2 \
  -o $OUT/prof_c3_gru_step_gemm$d $P --updates 1 > $OUT/prof_c3_gru_step_gemm$d.log 2>&1
done
ls -la $OUT
