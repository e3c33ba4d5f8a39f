#!/bin/bash
# C5 bench lines (cpu baseline + e2e) and the shard / chunk ncu at HEAD.
O=gpurun_out/c5f; mkdir -p $O
timeout 600 python bench.py --config C5 --steps 5 --warmup 5 > $O/bench_C5_1gpu.json 2> $O/C5.err
timeout 600 python bench.py --config C5 --emulate-gpus 8 --steps 10 --warmup 5 > $O/bench_C5_shard8.json 2> $O/C5s.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tt_wide" -c 1 -o $O/c5_shard_1m \
  python bench.py --config C5 --emulate-gpus 8 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/log_shard.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tt_wide" -c 1 -o $O/c5_chunk_1m \
  python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/log_chunk.txt 2>&1
ls -la $O
