#!/bin/bash
# Staged (cp.async) rank-code pre-pass vs the direct-load one on C2 / C4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prepass or special_thresholds or strategy_parity" 2>&1 | tail -3
tools/sweep2.sh C2 "HB_RC_STAGED=0" "HB_RC_STAGED=1" "HB_RC_STAGED=1,HB_RC_RB=2" "HB_RC_STAGED=1,HB_RC_RB=1" \
  "HB_RC_STAGED=1,HB_RC_SMEM_KB=24" "HB_RC_STAGED=1,HB_RC_SMEM_KB=96" "HB_RC_STAGED=1,HB_RC_SMEM_KB=96,HB_RC_RB=2" 2>&1
tools/sweep2.sh C4 "HB_RC_STAGED=0" "HB_RC_STAGED=1" 2>&1
for st in 0 1; do
HB_RC_STAGED=$st timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"rank_code|pttr" -c 2 --csv --log-file gpurun_out/c2_staged$st.csv \
  python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python - $st <<'PY'
import csv, sys
for r in csv.reader(open(f'gpurun_out/c2_staged{sys.argv[1]}.csv')):
    if len(r)>14 and 'kernel' in r[4]: print(sys.argv[1], r[4][:50], r[-1])
PY
done
