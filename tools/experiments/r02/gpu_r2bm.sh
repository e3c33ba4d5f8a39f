#!/bin/bash
# pre-pass table cap per CTA (HB_RC_SMEM_KB) with the row-word direct kernel: C4' and C2
O=gpurun_out/r2bm
mkdir -p $O
for kb in 48 64 96 32; do
  HB_RC_SMEM_KB=$kb timeout 900 python bench.py --config C4p --no-e2e --no-cpu >> $O/c4p_kb$kb.json 2>> $O/c4p_kb$kb.err
  HB_RC_SMEM_KB=$kb timeout 900 python bench.py --config C2 --no-e2e --no-cpu >> $O/c2_kb$kb.json 2>> $O/c2_kb$kb.err
done
du -sh $O
