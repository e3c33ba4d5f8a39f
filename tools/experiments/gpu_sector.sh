#!/bin/bash
# Sector-paired TT records for tt_wide_kernel: parity + C5 shard timing.
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tt_wide or tt_sector or c5_shard" 2>&1 | tail -3
for sec in 0 1; do
  HB_TT_SECTOR=$sec timeout 600 python bench.py --config C5 --rows 100000 --emulate-gpus 8 --steps 10 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sector=$sec', round(d['value']/1e6,2), 'Mrows/s', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3))"
done
HB_TT_SECTOR=1 timeout 600 python bench.py --config C5 --rows 100000 --steps 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('full 10k sector=1', round(d['value']/1e6,2), 'Mrows/s', round(d['ms_per_step'],3))"
