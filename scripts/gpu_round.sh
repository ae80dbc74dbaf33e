#!/usr/bin/env bash
# One gpurun call: GPU tests, smoke, bench, launch list, ncu captures.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_round.sh [tag]'
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu >> $OUT/nproc.txt 2>&1
( timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 ) > $OUT/pytest_gpu.log
echo "pytest rc=${PIPESTATUS[0]}"; tail -3 $OUT/pytest_gpu.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20 ) > $OUT/smoke.log
tail -2 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; cat $OUT/bench.json; tail -5 $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2>>$OUT/bench.err
cat $OUT/bench_ref.json
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python scripts/profile_update.py --updates 2 > $OUT/launches.log 2>&1
python scripts/launches.py $OUT/launches.csv 0.5 30 > $OUT/launches_summary.txt 2>&1
cat $OUT/launches_summary.txt
for k in gru_bwd_ks gru_fwd_ks; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
  -o $OUT/prof_$k python scripts/profile_update.py --updates 1 > $OUT/prof_$k.log 2>&1
done
for d in 0 1; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:gru_step_gemm_kernel<.{0,5}$d>" -s 2 -c 1 \
  -o $OUT/prof_gru_step_gemm$d python scripts/profile_update.py --updates 1 > $OUT/prof_gru_step_gemm$d.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 20 -c 2 \
  -o $OUT/prof_tc_gemm python scripts/profile_update.py --updates 1 > $OUT/prof_tc_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gae_scan|gather_tiled" -c 3 \
  -o $OUT/prof_gae_gather python scripts/profile_c5.py 24 > $OUT/prof_gae_gather.log 2>&1
fi
ls -la $OUT
