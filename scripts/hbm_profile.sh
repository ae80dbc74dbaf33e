#!/usr/bin/env bash
# ncu --set full of the HBM-bound kernels at C3 (configs[2]): close_rollout
# compaction (scatter, seq ids, descriptors + h0), the fused PPO loss, Adam.
#   gpurun -- 'bash scripts/hbm_profile.sh <tag>'
set -u
OUT=gpurun_out/${1:-hbm}
mkdir -p $OUT
P="python scripts/profile_update.py --N 4096 --epochs 3 --updates 1"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:compact_scatter|seq_ids|seq_desc" -c 3 \
  -o $OUT/prof_compaction $P > $OUT/prof_compaction.log 2>&1; echo "compaction rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:ppo_loss_rows|adam_kernel" -s 2 -c 3 \
  -o $OUT/prof_loss $P > $OUT/prof_loss.log 2>&1; echo "loss rc=$?"
