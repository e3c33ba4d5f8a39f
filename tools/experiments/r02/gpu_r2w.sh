#!/bin/bash
# two-level 32-B TT records (HB_TT_REC32): parity, C5 A/B, sanitizers, ncu
O=gpurun_out/r2w
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "tt_wide or c5 or auto_layout or auto_strategy or tree_chunks or strategy_parity" > $O/pytest_sel.txt 2>&1
for v in 1 0 1 0; do HB_TT_REC32=$v timeout 600 python bench.py --config C5 --emulate-gpus 8 --no-e2e --no-cpu >> $O/c5s_rec$v.json 2>> $O/c5s_rec$v.err; done
for v in 1 0; do HB_TT_REC32=$v timeout 900 python bench.py --config C5 --no-e2e --no-cpu >> $O/c5_rec$v.json 2>> $O/c5_rec$v.err; done
HB_TT_REC32=1 timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C5s python tools/one_call.py C5 --emulate-gpus 8 > $O/tr_C5s.log 2>&1
ncu -i /tmp/tr_C5s.ncu-rep --page raw --csv > $O/tr_C5s.raw.csv 2>/dev/null
ncu -i /tmp/tr_C5s.ncu-rep --page source --csv -k regex:tt_wide > $O/tr_C5s.source.csv 2>/dev/null
du -sh $O
