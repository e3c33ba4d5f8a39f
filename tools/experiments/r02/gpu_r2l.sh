#!/bin/bash
O=gpurun_out/r2l
mkdir -p $O
(timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "prepass or rank or one_kernel" 2>&1 | tail -3) > $O/pytest.txt 2>&1
timeout 900 python bench.py --no-e2e --no-cpu > $O/bench_C3.json 2> $O/bench_C3.err
for c in C4; do timeout 900 python bench.py --config $c --no-e2e --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; done
HB_RC_ONEK=0 timeout 900 python bench.py --config C4 --no-e2e --no-cpu > $O/bench_C4_staged.json 2> $O/bench_C4_staged.err
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -k regex:rank_code -o /tmp/tr_C3 python tools/one_call.py C3 > $O/tr_C3.log 2>&1
ncu -i /tmp/tr_C3.ncu-rep --page raw --csv > $O/tr_C3.raw.csv 2>/dev/null
