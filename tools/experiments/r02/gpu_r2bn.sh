#!/bin/bash
# C4 pre-pass table cap per CTA (HB_RC_SMEM_KB): 2-feature groups at 96 / 128 KB; direct vs staged
O=gpurun_out/r2bn
mkdir -p $O
for kb in 48 96 128; do HB_RC_SMEM_KB=$kb timeout 900 python bench.py --config C4 --no-e2e --no-cpu >> $O/c4_kb$kb.json 2>> $O/c4_kb$kb.err; done
for st in 0 1; do HB_RC_SMEM_KB=96 HB_RC_STAGED=$st timeout 900 python bench.py --config C4 --no-e2e --no-cpu >> $O/c4_kb96_st$st.json 2>> $O/c4_kb96_st$st.err; done
du -sh $O
