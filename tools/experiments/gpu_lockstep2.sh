#!/bin/bash
# Staged pre-pass with lockstep searches vs direct; ncu of both on C2.
O=gpurun_out/ls2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prepass" 2>&1 | tail -2
tools/sweep2.sh C2 "HB_RC_STAGED=0" "HB_RC_STAGED=1" "HB_RC_STAGED=1,HB_RC_RB=2" "HB_RC_STAGED=1,HB_RC_SMEM_KB=24" 2>&1
tools/sweep2.sh C4 "HB_RC_STAGED=0" "HB_RC_STAGED=1" 2>&1
for st in 0 1; do
HB_RC_STAGED=$st timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o $O/c2_rc$st \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
done
