#!/bin/bash
# AUTO after the pre-pass rule change; staged RB 2 vs 4 on C3 / C4 (repeated).
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prepass or auto_strategy or full_size" 2>&1 | tail -2
for rep in 1 2; do
tools/sweep2.sh C3 "HB_RC_RB=2" "HB_RC_RB=4" 2>&1
tools/sweep2.sh C4 "HB_RC_RB=2" "HB_RC_RB=4" 2>&1
done
tools/sweep2.sh C2 "HB_RANK_PRE=-1" 2>&1
tools/sweep2.sh C4p "HB_RANK_PRE=-1" 2>&1
