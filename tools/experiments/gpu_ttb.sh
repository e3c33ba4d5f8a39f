#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
  -k "tt_wide or tt_blocks or c5_shard or chain_trees or strategy_parity and tt" > gpurun_out/t_ttb.log 2>&1
tail -3 gpurun_out/t_ttb.log
for spec in "HB_TT_BLOCK=0" "HB_TT_BLOCK=1"; do
  out=$(env $spec timeout 300 python bench.py --config C5 --emulate-gpus 8 --steps 5 --no-e2e --no-cpu 2>&1 | tail -1)
  echo "$spec $(echo $out | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e6, "Mrows/s", d["ms_per_step"], "ms frac", d["roofline"]["frac"], d["roofline"]["kernel"])')"
done 2>&1 | tee gpurun_out/ttb_c5.txt
HB_PTT_RANK=1 HB_RANK_PRE=1 HB_RANK_CW=16 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"rank_code" -c 1 -o gpurun_out/rc_c2 \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out/rc_c2*
