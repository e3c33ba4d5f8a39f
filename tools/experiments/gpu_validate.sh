#!/bin/bash
O=gpurun_out/val
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
(time timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.err
