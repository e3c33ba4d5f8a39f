#!/bin/bash
# fp32 PTT (ptt_kernel) with interleaved warp units: parity + F8D3 AUTO A/B
O=gpurun_out/r2bd
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ptt or strategy_parity or feature_selection or edge_row or chain or checked or fuzz" > $O/pytest_sel.txt 2>&1
for v in 1 0 1 0; do HB_PTTR_INTERLEAVE=$v timeout 600 python bench.py --config F8D3 --no-e2e --no-cpu >> $O/f8_il$v.json 2>> $O/f8_il$v.err; done
du -sh $O
