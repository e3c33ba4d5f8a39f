#!/bin/bash
O=gpurun_out/r2i
mkdir -p $O
(timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "tt or c5 or TT" 2>&1 | tail -3) > $O/pytest_tt.txt 2>&1
timeout 900 python bench.py --no-e2e --no-cpu > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 python bench.py --config C5 --emulate-gpus 8 --no-e2e --no-cpu > $O/bench_C5s.json 2> $O/bench_C5s.err
timeout 900 python bench.py --config C5 --no-e2e --no-cpu > $O/bench_C5.json 2> $O/bench_C5.err
timeout 900 python bench.py --config F8D3 --strategy gemm --no-e2e > $O/bench_F8D3_gemm.json 2> $O/bench_F8D3_gemm.err
timeout 900 python bench.py --config F8D3 --no-e2e --no-cpu > $O/bench_F8D3_auto.json 2> $O/bench_F8D3_auto.err
for c in "tt" "tt-wide" "tt-wide-chunks" "tt-wide-multiclass" "ptt-rank-wrap" "ptt-fp32-wrap"; do
  timeout 900 compute-sanitizer --tool racecheck python tools/sanitize.py $c > $O/race_$c.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C3 python tools/one_call.py C3 > $O/tr_C3.log 2>&1
ncu -i /tmp/tr_C3.ncu-rep --page source --csv > $O/tr_C3.source.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_F8 python tools/one_call.py F8D3 > $O/tr_F8.log 2>&1
ncu -i /tmp/tr_F8.ncu-rep --page raw --csv > $O/tr_F8.raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C5s python tools/one_call.py C5 --emulate-gpus 8 > $O/tr_C5s.log 2>&1
ncu -i /tmp/tr_C5s.ncu-rep --page raw --csv > $O/tr_C5s.raw.csv 2>/dev/null
du -sh $O
