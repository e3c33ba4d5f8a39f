#!/bin/bash
# Evidence: full GPU suite + smoke, C4 (staged pre-pass AUTO) and C5 one-GPU (sector records) bench lines, ncu.
O=gpurun_out/evid4
mkdir -p $O
(time timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py --config C4 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --config C5 --rows 100000 --steps 5 --no-e2e > $O/bench_C5_1gpu.json 2> $O/bench_C5_1gpu.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file $O/launches_C4.csv \
  python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o $O/C4_rc \
  python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tt_wide" -c 1 -o $O/C5_1gpu_sector \
  python bench.py --config C5 --rows 100000 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
ls -la $O
