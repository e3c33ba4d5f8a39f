#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tt_wide or tt_blocks or c5_shard" 2>&1 | tail -1
HB_TTB_SYNC=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tt_wide or tt_blocks" 2>&1 | tail -1
for spec in "HB_TT_BLOCK=0" "HB_TTB_SYNC=0" "HB_TTB_SYNC=1"; do
  out=$(env $spec timeout 300 python bench.py --config C5 --emulate-gpus 8 --rows 100000 --steps 10 --no-e2e --no-cpu 2>&1 | tail -1)
  echo "$spec $(echo $out | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e6, "Mrows/s", d["ms_per_step"], "ms frac", d["roofline"]["frac"], d["roofline"]["kernel"], d["roofline"]["mean_levels_per_tree"])')"
done 2>&1 | tee gpurun_out/ttb_c5c.txt
tools/sweep2.sh C2 "HB_PTT_RANK=1,HB_RANK_PRE=1,HB_RANK_CW=32" "HB_PTT_RANK=1,HB_RANK_PRE=1,HB_RANK_CW=16"
HB_PTT_RANK=1 HB_RANK_PRE=1 HB_RANK_CW=16 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"rank_code|pttr" -c 2 --csv --log-file gpurun_out/c2_pre_launches3.csv \
  python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
