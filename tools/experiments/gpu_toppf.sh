#!/bin/bash
# tt_wide_kernel: L1 prefetch of the next tree group's top lines (HB_TT_TOP_PF).
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tt_wide or tt_sector" 2>&1 | tail -2
run() {
  env $1 timeout 600 python bench.py --config C5 --rows 100000 $2 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value']/1e6,2), 'Mrows/s', round(d['ms_per_step'],3), 'ms')"
}
for pf in 0 1; do run "HB_TT_TOP_PF=$pf" "--emulate-gpus 8 --steps 10"; done
for pf in 0 1; do run "HB_TT_TOP_PF=$pf" "--steps 3"; done
for pf in 0 1; do run "HB_TT_TOP_PF=$pf HB_TT_SECTOR=1" "--emulate-gpus 8 --steps 10"; done
