#!/bin/bash
# HEAD certification: full GPU suite (incl. the checked build), smoke, default bench
O=gpurun_out/r2ba
mkdir -p $O
(time timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.err
du -sh $O
