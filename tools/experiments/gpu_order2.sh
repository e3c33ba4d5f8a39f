#!/bin/bash
# Direct pre-pass with the group-major grid (HB_RC_ORDER=1) on C2; staged + order on C2.
HB_RC_ORDER=1 HB_RC_STAGED=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bucket_edges or degenerate" 2>&1 | tail -2
for rep in 1 2; do
tools/sweep2.sh C2 "HB_RC_ORDER=0" "HB_RC_ORDER=1" "HB_RC_STAGED=1" 2>&1
done
