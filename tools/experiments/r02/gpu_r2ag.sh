#!/bin/bash
# C2 with 32-bit code cells (two rows per lane, fewer warps) vs AUTO 16-bit; C3 row shards at the strong-scaling per-rank sizes
O=gpurun_out/r2ag
mkdir -p $O
for v in 32 0 32 0; do HB_RANK_CW=$v timeout 900 python bench.py --config C2 --no-e2e --no-cpu >> $O/c2_cw$v.json 2>> $O/c2_cw$v.err; done
for r in 5000000 2500000 1250000; do timeout 600 python bench.py --rows $r --no-e2e --no-cpu > $O/c3_rows$r.json 2> $O/c3_rows$r.err; done
du -sh $O
