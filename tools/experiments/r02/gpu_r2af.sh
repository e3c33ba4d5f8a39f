#!/bin/bash
# tt_wide_kernel with 6 / 8 walks per lane on 24 warps (launch bounds 768: 79-80 registers, no spill) vs 4 on 32
O=gpurun_out/r2af
mkdir -p $O
for g in 6 8 4 6 8 4; do HB_TT_G=$g timeout 600 python bench.py --config C5 --emulate-gpus 8 --no-e2e --no-cpu >> $O/c5s_g$g.json 2>> $O/c5s_g$g.err; done
HB_TT_G=6 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "tt_wide or c5_shard" > $O/pytest_g6.txt 2>&1
du -sh $O
