#!/bin/bash
# C4 pre-pass: table cap (SMEM vs global-memory tables) x staged / direct kernel.
tools/sweep2.sh C4 "HB_RC_STAGED=0" "HB_RC_STAGED=1" "HB_RC_STAGED=0,HB_RC_SMEM_KB=80" "HB_RC_STAGED=1,HB_RC_SMEM_KB=80" \
   "HB_RC_STAGED=0,HB_RC_SMEM_KB=100" "HB_RC_STAGED=1,HB_RC_SMEM_KB=100" "HB_RC_STAGED=1,HB_RC_RB=2" 2>&1
tools/sweep2.sh C2 "HB_RC_STAGED=-1" 2>&1
