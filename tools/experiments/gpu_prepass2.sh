#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
  -k "(strategy_parity and ptt) or special_thresholds or rank_prepass or depth_range" > gpurun_out/t_prepass.log 2>&1
tail -1 gpurun_out/t_prepass.log
for cfg in C2 C3; do
  tools/sweep2.sh $cfg "HB_PTT_RANK=1,HB_RANK_PRE=1,HB_RANK_CW=32" "HB_PTT_RANK=1,HB_RANK_PRE=1,HB_RANK_CW=16"
done 2>&1 | tee gpurun_out/sweep_prepass2.txt
HB_PTT_RANK=1 HB_RANK_PRE=1 HB_RANK_CW=16 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"rank_code|pttr" -c 6 --csv --log-file gpurun_out/c2_pre_launches.csv \
  python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
grep -o '"[a-z_]*kernel[^"]*","[^"]*","[^"]*","gpu__time_duration.sum","[^"]*","[^"]*"' gpurun_out/c2_pre_launches.csv | head; tail -4 gpurun_out/c2_pre_launches.csv | cut -c1-300
