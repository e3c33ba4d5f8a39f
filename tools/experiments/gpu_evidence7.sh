#!/bin/bash
O=gpurun_out/evid7
mkdir -p $O
(time timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5) > $O/pytest_gpu.txt 2>&1
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py --config C2 > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_C2.csv \
  python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o $O/C2_rc \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls $O
