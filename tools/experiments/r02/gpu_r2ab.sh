#!/bin/bash
# pttr_kernel register cap 80 (__maxnreg__, 800 threads x 80 = 64000 regs): C4 with two rows per lane; C2/C3/C4/C4' A/B
O=gpurun_out/r2ab
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "two_rows_per_lane or auto_layout or strategy_parity" > $O/pytest_sel.txt 2>&1
timeout 600 python bench.py --no-e2e --no-cpu >> $O/c3.json 2>> $O/c3.err
timeout 900 python bench.py --config C2 --no-e2e --no-cpu >> $O/C2.json 2>> $O/C2.err
timeout 900 python bench.py --config C4p --no-e2e --no-cpu >> $O/C4p.json 2>> $O/C4p.err
for v in 2 1; do HB_PTTR_RPL=$v timeout 900 python bench.py --config C4 --no-e2e --no-cpu >> $O/C4_rpl$v.json 2>> $O/C4_rpl$v.err; done
du -sh $O
