#!/bin/bash
# fp32 PTT X tiles by TMA bulk row copies + transpose (x_bulk): parity, F8D3 A/B, ncu
O=gpurun_out/r2z
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "x_bulk or strategy_parity or feature_selection or ptt_depth or special_thresholds or auto_layout or small_batch" > $O/pytest_sel.txt 2>&1
for v in -1 0 -1 0; do HB_X_BULK=$v timeout 600 python bench.py --config F8D3 --no-e2e --no-cpu >> $O/f8d3_bulk$v.json 2>> $O/f8d3_bulk$v.err; done
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_F8 python tools/one_call.py F8D3 > $O/tr_F8.log 2>&1
ncu -i /tmp/tr_F8.ncu-rep --page raw --csv > $O/tr_F8.raw.csv 2>/dev/null
ncu -i /tmp/tr_F8.ncu-rep --page source --csv -k regex:ptt_kernel > $O/tr_F8.source.csv 2>/dev/null
du -sh $O
