#!/bin/bash
# C3 staged pre-pass after branch-free searches: table cap (features per group) x rows per stage.
tools/sweep2.sh C3 "HB_RC_RB=2" "HB_RC_RB=4" "HB_RC_SMEM_KB=80,HB_RC_RB=2" "HB_RC_SMEM_KB=80,HB_RC_RB=4" "HB_RC_SMEM_KB=80,HB_RC_RB=1" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o gpurun_out/c3_st \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
