#!/bin/bash
# AUTO: 16-bit pair-load models group words for the direct row-word pre-pass (C4'): parity + C4' / C2 benches + ncu
O=gpurun_out/r2ar
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "rank_prepass or strategy_parity or full_size or prepass or auto_layout or one_kernel" > $O/pytest_sel.txt 2>&1
for c in C4p C2; do timeout 900 python bench.py --config $c --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C4p python tools/one_call.py C4p > $O/tr_C4p.log 2>&1
ncu -i /tmp/tr_C4p.ncu-rep --page raw --csv > $O/tr_C4p.raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C2 python tools/one_call.py C2 > $O/tr_C2.log 2>&1
ncu -i /tmp/tr_C2.ncu-rep --page raw --csv > $O/tr_C2.raw.csv 2>/dev/null
du -sh $O
