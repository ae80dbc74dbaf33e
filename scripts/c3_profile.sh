#!/usr/bin/env bash
# C3 launch list + ncu of the top GEMMs at C3 shapes (one gpurun call).
set -u
OUT=gpurun_out/${1:-r02a}
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 600 python scripts/profile_update.py --N 4096 --epochs 3 --updates 2 > $OUT/c3_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/c3_launches.csv python scripts/profile_update.py --N 4096 --epochs 3 --updates 2 > $OUT/c3_launches.log 2>&1
python scripts/launches.py $OUT/c3_launches.csv 0.5 40 > $OUT/c3_launches_summary.txt 2>&1
cat $OUT/c3_launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 40 -c 6 \
  -o $OUT/prof_c3_tc_gemm python scripts/profile_update.py --N 4096 --epochs 3 --updates 1 > $OUT/prof_c3_tc_gemm.log 2>&1

for d in 0 1; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:gru_step_gemm_kernel<.{0,5}$d>" -s 2 -c 1 \
  -o $OUT/prof_c3_gru_step_gemm$d python scripts/profile_update.py --N 4096 --epochs 3 --updates 1 > $OUT/prof_c3_gru_step_gemm$d.log 2>&1
done

ls -la $OUT
