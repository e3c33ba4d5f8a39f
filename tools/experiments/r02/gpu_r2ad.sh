#!/bin/bash
# two rows per lane with per-K accumulators (K <= 7: 7 fp64 sums per row, 2 trees in flight): C4 and C4' (pre-pass) A/B
O=gpurun_out/r2ad
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "two_rows_per_lane or auto_layout" > $O/pytest_sel.txt 2>&1
for v in 2 1; do HB_PTTR_RPL=$v timeout 900 python bench.py --config C4 --no-e2e --no-cpu >> $O/C4_rpl$v.json 2>> $O/C4_rpl$v.err; done
for v in 2 1; do HB_RANK_PRE=1 HB_PTTR_RPL=$v timeout 900 python bench.py --config C4p --no-e2e --no-cpu >> $O/C4p_pre_rpl$v.json 2>> $O/C4p_pre_rpl$v.err; done
timeout 900 python bench.py --config C4p --no-e2e --no-cpu >> $O/C4p_auto.json 2>> $O/C4p_auto.err
du -sh $O
