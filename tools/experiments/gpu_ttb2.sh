#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rank_prepass or special_thresholds" 2>&1 | tail -1
tools/sweep2.sh C2 "HB_PTT_RANK=1,HB_RANK_PRE=1,HB_RANK_CW=32" "HB_PTT_RANK=1,HB_RANK_PRE=1,HB_RANK_CW=16" 2>&1 | tee gpurun_out/sweep_prepass3.txt
HB_PTT_RANK=1 HB_RANK_PRE=1 HB_RANK_CW=16 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"rank_code|pttr" -c 4 --csv --log-file gpurun_out/c2_pre_launches2.csv \
  python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
cut -d, -f5,15 gpurun_out/c2_pre_launches2.csv | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ttb_kernel" -c 1 -o gpurun_out/ttb_c5 \
  python bench.py --config C5 --emulate-gpus 8 --rows 100000 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out/ttb_c5*
