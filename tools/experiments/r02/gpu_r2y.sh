#!/bin/bash
# wide-TT X tile fill: 8 independent 16-B loads per thread (indices recomputed, no spill); parity + C5 shard / full
O=gpurun_out/r2y
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "tt_wide or c5 or auto_layout or tree_chunks" > $O/pytest_sel.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --config C5 --emulate-gpus 8 --no-e2e --no-cpu >> $O/c5s.json 2>> $O/c5s.err; done
timeout 900 python bench.py --config C5 --no-e2e --no-cpu >> $O/c5.json 2>> $O/c5.err
du -sh $O
