#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tt_wide or c5_shard or chain_trees or graph_capture or streams" 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -8
for spec in "HB_TT_G=4"; do
  out=$(env $spec timeout 300 python bench.py --config C5 --emulate-gpus 8 --rows 100000 --steps 10 --no-e2e --no-cpu 2>&1 | tail -1)
  echo "$spec $(echo $out | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e6, "Mrows/s", d["ms_per_step"], "ms frac", d["roofline"]["frac"], d["roofline"]["kernel"])')"
done 2>&1 | tee gpurun_out/ttfin_c5.txt
