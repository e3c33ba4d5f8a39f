#!/bin/bash
# round 2 evidence: GPU suite, smoke, bench lines C1-C5, traffic captures, crossover, sanitizers
O=gpurun_out/r2h
mkdir -p $O
(time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.err
for c in C1 C2 C4 C4p; do timeout 900 python bench.py --config $c --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 python bench.py --config C5 --emulate-gpus 8 --no-e2e > $O/bench_C5s.json 2> $O/bench_C5s.err
timeout 900 python bench.py --config C5 --no-cpu > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
for spec in "C5 --emulate-gpus 8" "C5"; do
  tag=$(echo $spec | tr -d ' -')
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "hb_call/" -o /tmp/tr_$tag python tools/one_call.py $spec > $O/tr_$tag.log 2>&1
  ncu -i /tmp/tr_$tag.ncu-rep --page raw --csv > $O/tr_$tag.raw.csv 2>/dev/null
done
timeout 900 ncu --set full --clock-control none -k regex:gemm_tc -c 2 -o /tmp/gemm python tools/gemm_probe.py --only gemm > $O/gemm_ncu.log 2>&1
ncu -i /tmp/gemm.ncu-rep --page raw --csv > $O/gemm.raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $O/launches_C3.out 2>&1
timeout 1500 python tools/crossover.py --out $O/crossover.json > $O/crossover.txt 2>&1
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool python tools/sanitize.py > $O/san_$tool.txt 2>&1
done
du -sh $O
