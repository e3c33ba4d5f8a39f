#!/bin/bash
# C4' (RF, 7-wide class-distribution leaves): padded 16-B leaf loads vs packed
O=gpurun_out/r2r
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ptt or rank or C4 or c4" > $O/pytest_ptt.txt 2>&1
HB_PTTR_LEAF_VEC=0 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "C4p or c4p or rf" > $O/pytest_ptt_novec.txt 2>&1
for v in 1 0 1 0; do HB_PTTR_LEAF_VEC=$v timeout 600 python bench.py --config C4p --no-e2e --no-cpu >> $O/c4p_vec$v.json 2>> $O/c4p_vec$v.err; done
