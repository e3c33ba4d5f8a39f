#!/bin/bash
# tt_wide_kernel over pair-aligned BFS records with child lookahead (HB_TT_PAIR).
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tt_wide or tt_sector" 2>&1 | tail -2
run() {
  env $1 timeout 600 python bench.py --config C5 --rows 100000 $2 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value']/1e6,2), 'Mrows/s', round(d['ms_per_step'],3), 'ms')"
}
for rep in 1 2; do
for pr in 0 1; do run "HB_TT_PAIR=$pr" "--emulate-gpus 8 --steps 10"; done
done
run "HB_TT_PAIR=1 HB_TT_G=6" "--emulate-gpus 8 --steps 10"
