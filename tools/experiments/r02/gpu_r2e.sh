#!/bin/bash
# round 2: TT/C5 parity + C5 sweeps (walks per lane), GEMM probe + ncu, crossover with AUTO
O=gpurun_out/r2e
mkdir -p $O
(timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "tt or c5 or TT or leaf_values or single or chain or isolation or feature_selection or hand" 2>&1 | tail -5) > $O/pytest_tt.txt 2>&1
for g in 4 6 8; do HB_TT_G=$g timeout 600 python bench.py --config C5 --emulate-gpus 8 --no-e2e --no-cpu > $O/bench_C5s_g$g.json 2> $O/bench_C5s_g$g.err; done
timeout 900 python bench.py --config C5 --no-e2e --no-cpu > $O/bench_C5.json 2> $O/bench_C5.err
HB_TT_CHUNK=0 timeout 900 python bench.py --config C5 --no-e2e --no-cpu > $O/bench_C5_nochunk.json 2> $O/bench_C5_nochunk.err
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "hb_call/" -o /tmp/tr_C5s python tools/one_call.py C5 --emulate-gpus 8 > $O/tr_C5s.log 2>&1
ncu -i /tmp/tr_C5s.ncu-rep --page raw --csv > $O/tr_C5s.raw.csv 2>/dev/null
ncu -i /tmp/tr_C5s.ncu-rep --page source --csv > $O/tr_C5s.source.csv 2>/dev/null
timeout 900 python tools/gemm_probe.py > $O/gemm_probe.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 2 -o /tmp/gemm python tools/gemm_probe.py --only gemm > $O/gemm_ncu.log 2>&1
ncu -i /tmp/gemm.ncu-rep --page raw --csv > $O/gemm.raw.csv 2>/dev/null
ncu -i /tmp/gemm.ncu-rep --page source --csv > $O/gemm.source.csv 2>/dev/null
timeout 1500 python tools/crossover.py --out $O/crossover.json > $O/crossover.txt 2>&1
du -sh $O
