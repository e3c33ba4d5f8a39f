#!/bin/bash
run() {
  env $1 timeout 600 python bench.py --config C5 --rows 100000 $2 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value']/1e6,2), 'Mrows/s', round(d['ms_per_step'],3), 'ms', d['roofline']['layout'])"
}
for c in 2500 3336 4000 5000 6668 10000; do run "HB_TT_CHUNK=$c" "--steps 3"; done
for c in 2500 3336 5000; do run "HB_TT_CHUNK=$c HB_TT_SECTOR=0" "--steps 3 --rows 300000"; done
