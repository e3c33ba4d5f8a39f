#!/bin/bash
# round 2: GEMM v2 parity + probe + ncu; fp32 PTT D3/D5 ncu; crossover; C-config benches
O=gpurun_out/r2f
mkdir -p $O
(timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gemm or small or auto or strategy_parity or hand or single or chain or sixteen or more_outputs or leaf_values or c_consumer" 2>&1 | tail -8) > $O/pytest_sel.txt 2>&1
timeout 900 python tools/gemm_probe.py > $O/gemm_probe.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 1 -o /tmp/gemm python tools/gemm_probe.py --only gemm --trees 100 > $O/gemm_ncu.log 2>&1
ncu -i /tmp/gemm.ncu-rep --page raw --csv > $O/gemm.raw.csv 2>/dev/null
ncu -i /tmp/gemm.ncu-rep --page source --csv > $O/gemm.source.csv 2>/dev/null
for D in 3 5; do
timeout 900 ncu --set full --clock-control none -k regex:ptt_kernel -c 1 -o /tmp/ptt$D python tools/gemm_probe.py --only ptt --trees 100 --depth $D > $O/ptt${D}_ncu.log 2>&1
ncu -i /tmp/ptt$D.ncu-rep --page raw --csv > $O/ptt$D.raw.csv 2>/dev/null
done
timeout 1500 python tools/crossover.py --out $O/crossover.json > $O/crossover.txt 2>&1
timeout 900 python bench.py --no-cpu --no-e2e > $O/bench_C3.json 2> $O/bench_C3.err
for c in C2 C4 C4p; do timeout 900 python bench.py --config $c --no-e2e --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; done
du -sh $O
