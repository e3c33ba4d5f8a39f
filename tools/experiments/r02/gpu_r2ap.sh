#!/bin/bash
# row-word pre-pass with 5 row blocks per warp iteration for 10-row loads: parity + C2 A/B
O=gpurun_out/r2ap
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "rank_prepass or strategy_parity or full_size or prepass or two_rows or auto_layout" > $O/pytest_sel.txt 2>&1
for v in 1 0 1 0; do HB_RC_RW=$v timeout 900 python bench.py --config C2 --no-e2e --no-cpu >> $O/c2_rw$v.json 2>> $O/c2_rw$v.err; done
HB_RC_RW=1 timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C2 python tools/one_call.py C2 > $O/tr_C2.log 2>&1
ncu -i /tmp/tr_C2.ncu-rep --page raw --csv > $O/tr_C2.raw.csv 2>/dev/null
du -sh $O
