mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 400 python scripts/ab_bench.py "" "VER_REC_PERSIST=1" ""
