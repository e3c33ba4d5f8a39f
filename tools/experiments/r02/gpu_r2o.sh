#!/bin/bash
O=gpurun_out/r2o
mkdir -p $O
(HB_TT_REFILL=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "tt or c5 or TT" 2>&1 | tail -3) > $O/pytest_refill.txt 2>&1
for r in 0 1; do
  HB_TT_REFILL=$r timeout 600 python bench.py --config C5 --emulate-gpus 8 --no-e2e --no-cpu > $O/c5s_r$r.json 2> $O/c5s_r$r.err
done
HB_TT_REFILL=1 timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C5s python tools/one_call.py C5 --emulate-gpus 8 > $O/tr.log 2>&1
ncu -i /tmp/tr_C5s.ncu-rep --page raw --csv > $O/tr_C5s_refill.raw.csv 2>/dev/null
timeout 600 python tools/gemm_probe.py --trees 100 > $O/probe.txt 2>&1
