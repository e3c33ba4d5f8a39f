#!/bin/bash
# tt_wide_kernel: records below level L read through L2 only (ld.global.cg), keeping L1 for the top levels
O=gpurun_out/r2bl
mkdir -p $O
for v in 99 2 3 4 5 99 3 4; do HB_TT_L1_LEVELS=$v timeout 600 python bench.py --config C5 --emulate-gpus 8 --no-e2e --no-cpu >> $O/c5s_l$v.json 2>> $O/c5s_l$v.err; done
du -sh $O
