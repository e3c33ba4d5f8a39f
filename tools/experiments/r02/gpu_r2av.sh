#!/bin/bash
# pttr warp units interleaved over the grid (HB_PTTR_INTERLEAVE): parity + C2 / C3 / C3 1.25M / C4 / C4' A/B
O=gpurun_out/r2av
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ptt or prepass or full_size or two_rows or edge_row or strategy_parity or predict_host or events or graph or streams" > $O/pytest_sel.txt 2>&1
for v in 1 0; do
  HB_PTTR_INTERLEAVE=$v timeout 900 python bench.py --config C2 --no-e2e --no-cpu >> $O/c2_il$v.json 2>> $O/c2_il$v.err
  HB_PTTR_INTERLEAVE=$v timeout 600 python bench.py --no-e2e --no-cpu >> $O/c3_il$v.json 2>> $O/c3_il$v.err
  HB_PTTR_INTERLEAVE=$v timeout 600 python bench.py --rows 1250000 --no-e2e --no-cpu >> $O/c3s_il$v.json 2>> $O/c3s_il$v.err
  HB_PTTR_INTERLEAVE=$v timeout 900 python bench.py --config C4 --no-e2e --no-cpu >> $O/c4_il$v.json 2>> $O/c4_il$v.err
  HB_PTTR_INTERLEAVE=$v timeout 900 python bench.py --config C4p --no-e2e --no-cpu >> $O/c4p_il$v.json 2>> $O/c4p_il$v.err
done
du -sh $O
