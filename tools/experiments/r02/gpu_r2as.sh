#!/bin/bash
# C3 TMA pre-pass with twice the buckets per threshold (HB_RC_DENSITY=2: one fewer window step)
O=gpurun_out/r2as
mkdir -p $O
for v in 2 1 4 2 1; do HB_RC_DENSITY=$v timeout 600 python bench.py --no-e2e --no-cpu >> $O/c3_dens$v.json 2>> $O/c3_dens$v.err; done
du -sh $O
