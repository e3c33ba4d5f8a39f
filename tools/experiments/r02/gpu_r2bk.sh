#!/bin/bash
# bench line with seeds / layout / device-memory fields: contract tests + C3 / C5 shard lines
O=gpurun_out/r2bk
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider tests/test_bench_contract.py > $O/pytest_bench.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > $O/c3.json 2> $O/c3.err
timeout 600 python bench.py --config C5 --emulate-gpus 8 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/c5s.json 2> $O/c5s.err
du -sh $O
