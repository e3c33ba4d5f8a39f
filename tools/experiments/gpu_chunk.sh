#!/bin/bash
# TT over L2-resident tree chunks for models larger than L2 (HB_TT_CHUNK).
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tree_chunks or tt_wide or c5_full" 2>&1 | tail -2
run() {
  env $1 timeout 600 python bench.py --config C5 --rows 100000 $2 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value']/1e6,2), 'Mrows/s', round(d['ms_per_step'],3), 'ms', d['roofline']['layout'])"
}
for c in 0 -1 1000 1500 2500; do run "HB_TT_CHUNK=$c" "--steps 3"; done
run "HB_TT_CHUNK=-1" "--steps 3 --rows 1000000"
run "HB_TT_CHUNK=0" "--steps 3 --rows 1000000"
