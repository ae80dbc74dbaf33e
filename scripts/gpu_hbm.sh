#!/usr/bin/env bash
# GAE / gather iteration: parity tests of the scan and the gather, the C5 sweep
# point, ncu of both kernels at 2^26, and (optional) extra commands.
#   gpurun -- 'bash scripts/gpu_hbm.sh <tag>'
set -u
OUT=gpurun_out/${1:-hbm}
mkdir -p $OUT
( timeout 900 python -m pytest tests/test_golden.py tests/test_gpu_gae_stress.py tests/test_gpu_ragged.py \
    tests/test_gpu_parity.py tests/test_learner.py -x -q 2>&1 | tail -15 ) > $OUT/pytest.log
tail -3 $OUT/pytest.log
timeout 600 python scripts/sweep_c5.py > $OUT/c5.json 2> $OUT/c5.err; echo "c5 rc=$?"; cat $OUT/c5.json; tail -3 $OUT/c5.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gae_scan|gather_tiled" -c 3 \
  -o $OUT/prof_gae_gather python scripts/profile_c5.py 26 > $OUT/prof_gae_gather.log 2>&1
echo "ncu rc=$?"
fi
