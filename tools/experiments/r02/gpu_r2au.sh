#!/bin/bash
# row-word pre-pass: next four rows' X loaded before the current search (register double buffer): parity + C2 / C4' benches
O=gpurun_out/r2au
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "rank_prepass or strategy_parity or full_size or prepass" > $O/pytest_sel.txt 2>&1
for i in 1 2; do for c in C2 C4p; do timeout 900 python bench.py --config $c --no-e2e --no-cpu >> $O/bench_$c.json 2>> $O/bench_$c.err; done; done
du -sh $O
