#!/bin/bash
# AUTO: pre-pass with 16-bit cells for long walks (C4'): layout tests, C4' / C4 / C2 / C3 benches
O=gpurun_out/r2ae
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "auto_layout or full_size or strategy_parity or rank_prepass" > $O/pytest_sel.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
for c in C4p C4 C2; do timeout 900 python bench.py --config $c --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C4p python tools/one_call.py C4p > $O/tr_C4p.log 2>&1
ncu -i /tmp/tr_C4p.ncu-rep --page raw --csv > $O/tr_C4p.raw.csv 2>/dev/null
du -sh $O
