#!/bin/bash
# Round-1 pre-pass evaluation: parity of the rank-code pre-pass + layout sweep.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
  -k "(strategy_parity and ptt) or special_thresholds or rank_prepass or depth_range" > gpurun_out/t_prepass.log 2>&1
tail -3 gpurun_out/t_prepass.log
for cfg in C2 C3 C4 C4p; do
  tools/sweep2.sh $cfg "HB_RANK_PRE=0" "HB_PTT_RANK=1,HB_RANK_PRE=1,HB_RANK_CW=32" "HB_PTT_RANK=1,HB_RANK_PRE=1,HB_RANK_CW=16" \
    "HB_PTT_RANK=1,HB_RANK_PRE=1,HB_RANK_CW=16,HB_NW=16" "HB_PTT_RANK=1,HB_RANK_PRE=1,HB_RANK_CW=32,HB_NW=16"
done 2>&1 | tee gpurun_out/sweep_prepass.txt
