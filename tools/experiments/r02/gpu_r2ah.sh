#!/bin/bash
# rank-coded PTT launches trim consumer warps to fill the last round of row tiles (HB_NW_TRIM): parity + C2 / C3 shard A/B
O=gpurun_out/r2ai
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "edge_row or two_rows" > $O/pytest_sel.txt 2>&1
for v in 1 0; do HB_NW_TRIM=$v timeout 900 python bench.py --config C2 --no-e2e --no-cpu >> $O/c2_trim$v.json 2>> $O/c2_trim$v.err; done
for v in 1 0; do HB_NW_TRIM=$v timeout 600 python bench.py --rows 1250000 --no-e2e --no-cpu >> $O/c3_1250k_trim$v.json 2>> $O/c3_1250k_trim$v.err; done
for v in 1 0; do HB_NW_TRIM=$v timeout 600 python bench.py --rows 2500000 --no-e2e --no-cpu >> $O/c3_2500k_trim$v.json 2>> $O/c3_2500k_trim$v.err; done
du -sh $O
