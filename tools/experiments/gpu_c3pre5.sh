#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "staged_spans or bucket_edges" 2>&1 | tail -2
for rep in 1 2; do
tools/sweep2.sh C3 "HB_RC_RB=-1" "HB_RC_ONE=1,HB_RC_RB=2" "HB_RC_ONE=0,HB_RC_SMEM_KB=80,HB_RC_RB=2" "HB_RC_ONE=0,HB_RC_SMEM_KB=72,HB_RC_RB=2" "HB_RC_ONE=0,HB_RC_SMEM_KB=110,HB_RC_RB=2" 2>&1
done
tools/sweep2.sh C4 "HB_RC_RB=-1" "HB_RC_ONE=0,HB_RC_SMEM_KB=84,HB_RC_RB=2" 2>&1
