#!/bin/bash
# 32-B TT records: LDG.256 vs 2 x LDG.128 vs 16-B records on the C5 shard; source-level ncu of both record forms
O=gpurun_out/r2x
mkdir -p $O
for i in 1 2; do
  HB_TT_REC32=1 HB_TT_REC32_LD128=1 timeout 600 python bench.py --config C5 --emulate-gpus 8 --no-e2e --no-cpu >> $O/c5s_ld128.json 2>> $O/c5s_ld128.err
  HB_TT_REC32=1 timeout 600 python bench.py --config C5 --emulate-gpus 8 --no-e2e --no-cpu >> $O/c5s_ld256.json 2>> $O/c5s_ld256.err
  HB_TT_REC32=0 timeout 600 python bench.py --config C5 --emulate-gpus 8 --no-e2e --no-cpu >> $O/c5s_rec16.json 2>> $O/c5s_rec16.err
done
for v in 0 1; do
  HB_TT_REC32=$v timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C5s_$v python tools/one_call.py C5 --emulate-gpus 8 > $O/tr_C5s_$v.log 2>&1
  ncu -i /tmp/tr_C5s_$v.ncu-rep --page raw --csv > $O/tr_C5s_$v.raw.csv 2>/dev/null
  ncu -i /tmp/tr_C5s_$v.ncu-rep --page source --csv -k regex:tt_wide > $O/tr_C5s_$v.source.csv 2>/dev/null
done
du -sh $O
