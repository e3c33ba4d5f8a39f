#!/bin/bash
O=gpurun_out/evid8
mkdir -p $O
(time timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5) > $O/pytest_gpu.txt 2>&1
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 python bench.py --config C2 > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 python bench.py --config C4 > $O/bench_C4.json 2> $O/bench_C4.err
ls $O
