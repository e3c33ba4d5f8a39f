#!/bin/bash
O=gpurun_out/evid2
mkdir -p $O
timeout 900 python bench.py --config C4 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --config C1 --no-e2e > $O/bench_C1.json 2> $O/bench_C1.err
timeout 900 python bench.py --config C5 --rows 100000 --steps 5 --no-e2e > $O/bench_C5_1gpu.json 2> $O/bench_C5_1gpu.err
timeout 900 python bench.py --config C5 --rows 100000 --emulate-gpus 8 --steps 10 --no-e2e --no-cpu > $O/bench_C5_shard8.json 2> $O/bench_C5_shard8.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tt_wide" -c 1 -o $O/C5_shard_tt \
  python bench.py --config C5 --rows 100000 --emulate-gpus 8 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pttr_kernel" -c 1 -o $O/C4_pttr \
  python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py > $O/san_$tool.txt 2>&1
  tail -2 $O/san_$tool.txt
done
ls -la $O
