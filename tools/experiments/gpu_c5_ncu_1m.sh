#!/bin/bash
# C5 at its 1M-row bench default: ncu --set full of one tt_wide_kernel launch
# (1/8 tree shard; all 10k trees = first L2 chunk) + the launch list of the
# all-trees step. Reports in gpurun_out/c5n/.
O=gpurun_out/c5n; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tt_wide" -c 1 -o $O/c5_shard_1m \
  python bench.py --config C5 --emulate-gpus 8 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/log_shard.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tt_wide" -c 1 -o $O/c5_chunk_1m \
  python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/log_chunk.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_C5.csv \
  python bench.py --config C5 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la $O
