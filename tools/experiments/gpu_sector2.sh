#!/bin/bash
# Sector-paired TT records with BFS top levels: parity + C5 shard / full timing per top depth.
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tt_wide or tt_sector or c5_shard" 2>&1 | tail -3
run() {
  env $1 timeout 600 python bench.py --config C5 --rows 100000 $2 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value']/1e6,2), 'Mrows/s', round(d['ms_per_step'],3), 'ms')"
}
for top in 0 3 4 5 6; do run "HB_TT_SECTOR=1 HB_TT_SECTOR_TOP=$top" "--emulate-gpus 8 --steps 10"; done
run "HB_TT_SECTOR=0" "--emulate-gpus 8 --steps 10"
for top in 4 6; do run "HB_TT_SECTOR=1 HB_TT_SECTOR_TOP=$top" "--steps 3"; done
run "HB_TT_SECTOR=0" "--steps 3"
