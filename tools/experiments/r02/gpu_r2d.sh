#!/bin/bash
# round 2: GPU suite, bench lines, per-call ncu traffic (reports kept in /tmp,
# only CSV exports come back), launch list
O=gpurun_out/r2d
mkdir -p $O
(time timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -40) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.err
for c in C2 C4 C4p C1; do timeout 900 python bench.py --config $c --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 python bench.py --config C5 --emulate-gpus 8 --no-e2e > $O/bench_C5s.json 2> $O/bench_C5s.err
timeout 900 python bench.py --config C5 --no-e2e --no-cpu > $O/bench_C5.json 2> $O/bench_C5.err
for spec in "C3" "C2" "C4" "C4p" "C5 --emulate-gpus 8" "C5"; do
  tag=$(echo $spec | tr -d ' -')
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "hb_call/" -o /tmp/tr_$tag python tools/one_call.py $spec > $O/tr_$tag.log 2>&1
  ncu -i /tmp/tr_$tag.ncu-rep --page raw --csv > $O/tr_$tag.raw.csv 2>/dev/null
  ncu -i /tmp/tr_$tag.ncu-rep --page details > $O/tr_$tag.details.txt 2>/dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $O/launches_C3.out 2>&1
du -sh $O
