set -u
OUT=gpurun_out/r02q
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
( timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 ) > $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 ) > $OUT/smoke.log
tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; head -c 600 $OUT/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2>>$OUT/bench.err
head -c 600 $OUT/bench_ref.json
timeout 900 python scripts/configs_table.py > $OUT/configs_table.jsonl 2> $OUT/configs_table.err
cat $OUT/configs_table.jsonl
