#!/bin/bash
# Direct pre-pass with lockstep searches: parity + C2 / C4 timing + launch split.
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prepass or special_thresholds or strategy_parity or full_size" 2>&1 | tail -3
tools/sweep2.sh C2 "HB_RC_STAGED=-1" "HB_RC_SMEM_KB=24" "HB_RC_SMEM_KB=96" 2>&1
tools/sweep2.sh C4 "HB_RC_STAGED=0" "HB_RC_STAGED=1" "HB_RC_STAGED=0,HB_RC_SMEM_KB=80" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"rank_code|pttr" -c 2 --csv --log-file gpurun_out/c2_lock.csv \
  python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
for r in csv.reader(open('gpurun_out/c2_lock.csv')):
    if len(r)>14 and 'kernel' in r[4]: print(r[4][:50], r[-1])
PY
