#!/bin/bash
# round 2: GPU suite + smoke + C3/C4/C5-shard bench after the fp64 accumulator change
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
(time timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -25) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py --no-cpu > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 python bench.py --no-cpu --no-e2e --config C4 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --no-cpu --no-e2e --config C2 > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 python bench.py --no-cpu --no-e2e --config C5 --emulate-gpus 8 > $O/bench_C5s.json 2> $O/bench_C5s.err
