#!/bin/bash
# C3 scorer launch shape with pre-pass codes: warps, ring stages, chunk size.
python - <<'PY'
import synth, paper_2010_04804_b200 as hb
c, e = synth.make_config("C3")
m = hb.Model(e, device=0)
print({k: m.info[k] for k in ("kernel_name", "rank_prepass", "code_cell_bits", "rows_per_cta", "tree_stride_bytes")})
PY
tools/sweep2.sh C3 "HB_NW=-1" "HB_CH=16" "HB_CH=24" "HB_CH=48" "HB_NS=3" "HB_NS=3,HB_CH=16" "HB_NW=16" "HB_PREFETCH=0" 2>&1
