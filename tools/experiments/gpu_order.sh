#!/bin/bash
# Staged pre-pass grid order: group-major with contiguous row slices (HB_RC_ORDER=1).
HB_RC_ORDER=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "staged_spans or bucket_edges or degenerate" 2>&1 | tail -2
for rep in 1 2; do
tools/sweep2.sh C3 "HB_RC_ORDER=0" "HB_RC_ORDER=1" 2>&1
done
tools/sweep2.sh C4 "HB_RC_ORDER=0" "HB_RC_ORDER=1" 2>&1
HB_RC_ORDER=1 timeout 600 ncu --set full --clock-control none -k regex:"rank_code" -c 1 -o gpurun_out/c3_ord \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
