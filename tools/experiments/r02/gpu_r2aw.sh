#!/bin/bash
# round 2 final evidence refresh 3 (interleaved warp units, pre-pass X double buffer)
O=gpurun_out/r2aw
mkdir -p $O
nproc > $O/nproc.txt
(time timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_C3.json 2> $O/bench_C3.err
for c in C1 C2 C4 C4p; do timeout 900 python bench.py --config $c --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 python bench.py --config C5 --emulate-gpus 8 --no-e2e > $O/bench_C5s.json 2> $O/bench_C5s.err
timeout 900 python bench.py --config C5 --no-cpu > $O/bench_C5.json 2> $O/bench_C5.err
timeout 900 python bench.py --config F8D3 --strategy gemm --no-e2e > $O/bench_F8D3_gemm.json 2> $O/bench_F8D3_gemm.err
timeout 900 python bench.py --config F8D3 --no-e2e > $O/bench_F8D3_auto.json 2> $O/bench_F8D3_auto.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
for spec in C3 C2 C4 C4p; do
  timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_$spec python tools/one_call.py $spec > $O/tr_$spec.log 2>&1
  ncu -i /tmp/tr_$spec.ncu-rep --page raw --csv > $O/tr_$spec.raw.csv 2>/dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $O/launches_C3.out 2>&1
du -sh $O
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C5s python tools/one_call.py C5 --emulate-gpus 8 > $O/tr_C5s.log 2>&1
ncu -i /tmp/tr_C5s.ncu-rep --page raw --csv > $O/tr_C5s.raw.csv 2>/dev/null
du -sh $O
