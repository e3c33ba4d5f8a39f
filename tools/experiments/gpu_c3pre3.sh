#!/bin/bash
# C3 pre-pass (staged, single-feature groups): rows per stage, table cap; ncu of the pre-pass.
tools/sweep2.sh C3 "HB_RANK_PRE=1" "HB_RANK_PRE=1,HB_RC_RB=2" "HB_RANK_PRE=1,HB_RC_RB=1" "HB_RANK_PRE=1,HB_RC_SMEM_KB=36" "HB_RANK_PRE=1,HB_RC_SMEM_KB=36,HB_RC_RB=1" 2>&1
HB_RANK_PRE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o gpurun_out/c3_rc \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
