#!/bin/bash
# Refresh every config's bench line at HEAD (results in gpurun_out/rb/).
O=gpurun_out/rb; mkdir -p $O
timeout 300 python bench.py --config C1 > $O/bench_C1.json 2> $O/C1.err
timeout 300 python bench.py --config C2 > $O/bench_C2.json 2> $O/C2.err
timeout 400 python bench.py --config C4 > $O/bench_C4.json 2> $O/C4.err
timeout 300 python bench.py --config C4p > $O/bench_C4p.json 2> $O/C4p.err
timeout 600 python bench.py --config C5 --steps 5 --warmup 5 > $O/bench_C5_1gpu.json 2> $O/C5.err
timeout 600 python bench.py --config C5 --emulate-gpus 8 --steps 10 --warmup 5 > $O/bench_C5_shard8.json 2> $O/C5s.err
