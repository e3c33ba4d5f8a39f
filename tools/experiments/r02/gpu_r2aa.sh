#!/bin/bash
# pttr_kernel with two rows per lane (HB_PTTR_RPL=2): parity, C3 / C2 / C4 A/B, ncu
O=gpurun_out/r2aa
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "two_rows_per_lane or auto_layout or full_size" > $O/pytest_sel.txt 2>&1
for v in 2 1 2 1; do HB_PTTR_RPL=$v timeout 600 python bench.py --no-e2e --no-cpu >> $O/c3_rpl$v.json 2>> $O/c3_rpl$v.err; done
for c in C2 C4; do for v in 2 1; do HB_PTTR_RPL=$v timeout 900 python bench.py --config $c --no-e2e --no-cpu >> $O/${c}_rpl$v.json 2>> $O/${c}_rpl$v.err; done; done
HB_PTTR_RPL=2 timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C3r2 python tools/one_call.py C3 > $O/tr_C3r2.log 2>&1
ncu -i /tmp/tr_C3r2.ncu-rep --page raw --csv > $O/tr_C3r2.raw.csv 2>/dev/null
du -sh $O
