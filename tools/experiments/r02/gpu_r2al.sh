#!/bin/bash
# C4 two rows per lane (class-sum flushes) with 16-bit cells (24 warps) vs one row with 32-bit cells
O=gpurun_out/r2al
mkdir -p $O
for i in 1 2; do
HB_RANK_CW=16 HB_PTTR_RPL=2 timeout 900 python bench.py --config C4 --no-e2e --no-cpu >> $O/C4_cw16_rpl2.json 2>> $O/C4_cw16_rpl2.err
HB_RANK_CW=16 HB_PTTR_RPL=1 timeout 900 python bench.py --config C4 --no-e2e --no-cpu >> $O/C4_cw16_rpl1.json 2>> $O/C4_cw16_rpl1.err
done
du -sh $O
