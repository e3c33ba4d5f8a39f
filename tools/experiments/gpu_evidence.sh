#!/bin/bash
# Round evidence: full GPU test suite, smoke, per-config bench lines, the
# reference arm, launch lists and ncu --set full captures of the top kernels.
# Results land in gpurun_out/evid/ (copied into profiles/ afterwards).
O=gpurun_out/evid
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
(time timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.err
for c in C1 C2 C4 C4p; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config C5 --rows 100000 --steps 5 --no-e2e > $O/bench_C5_1gpu.json 2> $O/bench_C5_1gpu.err
timeout 900 python bench.py --config C5 --rows 100000 --emulate-gpus 8 --steps 10 --no-e2e --no-cpu > $O/bench_C5_shard8.json 2> $O/bench_C5_shard8.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/reference_C3.json 2> $O/reference_C3.err
# launch lists (cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_C3.csv \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_C2.csv \
  python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
# full captures of the dominant kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pttr_kernel" -c 1 -o $O/C3_pttr \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rank_code|pttr_kernel" -c 2 -o $O/C2_pre \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la $O
