#!/bin/bash
# TMA pre-pass with the fixed-window search: parity, C3, sanitizers, ncu
O=gpurun_out/r2t
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "tma or prepass or rank_code or auto_layout or full_size or ptt_depth or special_thresholds or events" > $O/pytest_sel.txt 2>&1
for v in 1 1; do HB_RC_TMA=$v timeout 600 python bench.py --no-e2e --no-cpu >> $O/c3_tma$v.json 2>> $O/c3_tma$v.err; done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py ptt-rank-prepass-tma-32 ptt-rank-prepass-tma-16 ptt-rank-prepass-32 ptt-rank-wrap > $O/san_$tool.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C3 python tools/one_call.py C3 > $O/tr_C3.log 2>&1
ncu -i /tmp/tr_C3.ncu-rep --page raw --csv > $O/tr_C3.raw.csv 2>/dev/null
ncu -i /tmp/tr_C3.ncu-rep --page source --csv -k regex:rank_code_tma > $O/tr_C3_tma.source.csv 2>/dev/null
du -sh $O
