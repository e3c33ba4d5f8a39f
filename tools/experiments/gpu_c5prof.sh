#!/bin/bash
O=gpurun_out/c5p
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tt_wide" -c 1 -o $O/c5_shard \
  python bench.py --config C5 --rows 100000 --emulate-gpus 8 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/log.txt 2>&1
ls -la $O
