#!/bin/bash
# Evidence after the pre-pass changes: bench lines C2 / C4, launch lists, ncu of the pre-pass kernels.
O=gpurun_out/evid3
mkdir -p $O
timeout 900 python bench.py --config C2 > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 python bench.py --config C4 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_C2.csv \
  python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file $O/launches_C4.csv \
  python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o $O/C2_rc \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o $O/C4_rc \
  python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
ls -la $O
