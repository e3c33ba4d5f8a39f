#!/bin/bash
# HEAD certification 3: full GPU suite, smoke, default bench, F8D3 AUTO line
O=gpurun_out/r2bg
mkdir -p $O
(time timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 python bench.py --config F8D3 --no-e2e > $O/bench_F8D3_auto.json 2> $O/bench_F8D3_auto.err
du -sh $O
