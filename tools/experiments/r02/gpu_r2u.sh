#!/bin/bash
# fixed-window search in every pre-pass kernel: parity + C2 / C3 / C4 benches
O=gpurun_out/r2u
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "tma or prepass or rank_code or auto_layout or full_size or ptt_depth or special_thresholds or deep_bucket or strategy_parity" > $O/pytest_sel.txt 2>&1
timeout 600 python bench.py --no-e2e --no-cpu > $O/c3.json 2> $O/c3.err
for c in C2 C4; do timeout 900 python bench.py --config $c --no-e2e --no-cpu > $O/$c.json 2> $O/$c.err; done
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py ptt-rank-prepass-32 ptt-rank-prepass-16 ptt-rank-prepass-staged-16 ptt-rank-prepass-staged-32-rb1 ptt-rank-prepass-column ptt-rank-prepass-rows8 > $O/san_$tool.txt 2>&1
done
du -sh $O
