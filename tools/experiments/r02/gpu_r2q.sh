#!/bin/bash
O=gpurun_out/r2q
mkdir -p $O
(time timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
for rows in 5000000 2500000 1250000; do timeout 600 python bench.py --rows $rows --no-e2e --no-cpu > $O/c3_rows$rows.json 2> $O/c3_rows$rows.err; done
timeout 900 python bench.py --config F8D3 --strategy gemm --no-e2e --no-cpu > $O/bench_F8D3_gemm.json 2> $O/bench_F8D3_gemm.err
timeout 900 python bench.py --config F8D3 --no-e2e --no-cpu > $O/bench_F8D3_auto.json 2> $O/bench_F8D3_auto.err
