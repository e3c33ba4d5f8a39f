#!/bin/bash
# C4' pre-pass: multi-word groups + direct row-word kernel (HB_RC_ONEK_MAX_GROUPS=0) vs the column kernel; C3 likewise
O=gpurun_out/r2aq
mkdir -p $O
for v in 0 32 0 32; do HB_RC_ONEK_MAX_GROUPS=$v timeout 900 python bench.py --config C4p --no-e2e --no-cpu >> $O/c4p_onek$v.json 2>> $O/c4p_onek$v.err; done
for v in 0 32; do HB_RC_ONEK_MAX_GROUPS=$v timeout 900 python bench.py --config C4 --no-e2e --no-cpu >> $O/c4_onek$v.json 2>> $O/c4_onek$v.err; done
HB_RC_ONEK_MAX_GROUPS=0 timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C4p python tools/one_call.py C4p > $O/tr_C4p.log 2>&1
ncu -i /tmp/tr_C4p.ncu-rep --page raw --csv > $O/tr_C4p.raw.csv 2>/dev/null
du -sh $O
