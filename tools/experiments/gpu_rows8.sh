#!/bin/bash
# Direct pre-pass: 4 vs 8 row blocks per batch (8 vs 16 lockstep searches per lane).
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prepass" 2>&1 | tail -2
tools/sweep2.sh C2 "HB_RC_ROWS=4" "HB_RC_ROWS=8" "HB_RC_ROWS=8,HB_RC_SMEM_KB=64" "HB_RC_ROWS=4,HB_RC_SMEM_KB=40" 2>&1
tools/sweep2.sh C4 "HB_RC_STAGED=0,HB_RC_ROWS=8" "HB_RC_STAGED=0,HB_RC_ROWS=8,HB_RC_SMEM_KB=80" 2>&1
