#!/bin/bash
# Branch-free lockstep searches: every pre-pass kernel on C2 / C3 / C4.
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prepass" 2>&1 | tail -2
tools/sweep2.sh C3 "HB_RANK_PRE=-1" "HB_RANK_PRE=1" "HB_RANK_PRE=1,HB_RC_STAGED=1,HB_RC_RB=2" "HB_RANK_PRE=1,HB_RC_STAGED=1" "HB_RANK_PRE=1,HB_RC_STAGED=0" 2>&1
tools/sweep2.sh C2 "HB_RANK_PRE=-1" "HB_RC_STAGED=0" "HB_RC_STAGED=1" 2>&1
tools/sweep2.sh C4 "HB_RANK_PRE=-1" "HB_RC_STAGED=0" 2>&1
tools/sweep2.sh C4p "HB_RANK_PRE=-1" "HB_RANK_PRE=1" 2>&1
