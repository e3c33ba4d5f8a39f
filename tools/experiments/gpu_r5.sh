#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rank_prepass or special_thresholds or depth_range or (strategy_parity and ptt) or tt_wide" 2>&1 | tail -1
HB_TT_G=8 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tt_wide or c5_shard" 2>&1 | tail -1
tools/sweep2.sh C2 "HB_RANK_PRE=-1" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"rank_code|pttr" -c 2 --csv --log-file gpurun_out/c2_pre_launches4.csv \
  python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
for r in csv.reader(open('gpurun_out/c2_pre_launches4.csv')):
    if len(r)>14 and 'kernel' in r[4]: print(r[4][:40], r[-1])
PY
for spec in "HB_TT_G=4" "HB_TT_G=6" "HB_TT_G=8"; do
  out=$(env $spec timeout 300 python bench.py --config C5 --emulate-gpus 8 --rows 100000 --steps 10 --no-e2e --no-cpu 2>&1 | tail -1)
  echo "$spec $(echo $out | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e6, "Mrows/s", d["ms_per_step"], "ms frac", d["roofline"]["frac"], d["roofline"]["kernel"])')"
done 2>&1 | tee gpurun_out/ttg_c5.txt
