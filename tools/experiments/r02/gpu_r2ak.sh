#!/bin/bash
# two rows per lane for per-class scalar trees via class-sum flushes (C4): parity + C4 A/B
O=gpurun_out/r2ak
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "two_rows_per_lane or events or auto_layout" > $O/pytest_sel.txt 2>&1
for v in 2 1 2 1; do HB_PTTR_RPL=$v timeout 900 python bench.py --config C4 --no-e2e --no-cpu >> $O/C4_rpl$v.json 2>> $O/C4_rpl$v.err; done
du -sh $O
