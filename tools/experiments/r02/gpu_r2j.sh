#!/bin/bash
O=gpurun_out/r2j
mkdir -p $O
(timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "ptt or tt or strategy or prepass or rank or small or graph or streams" 2>&1 | tail -3) > $O/pytest.txt 2>&1
timeout 900 python bench.py --no-e2e --no-cpu > $O/bench_C3.json 2> $O/bench_C3.err
for c in C2 C4 C4p; do timeout 900 python bench.py --config $c --no-e2e --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in tt ptt-rank-wrap ptt-fp32-wrap ptt-rank ptt-fp32 ptt-rank-prepass-32 ptt-rank-prepass-staged-16; do
  timeout 900 compute-sanitizer --tool racecheck python tools/sanitize.py $c > $O/race_$c.txt 2>&1
done
