#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tt_wide or tt_blocks or c5_shard" 2>&1 | tail -1
for spec in "HB_TT_BLOCK=0" "HB_TT_BLOCK=1"; do
  out=$(env $spec timeout 300 python bench.py --config C5 --emulate-gpus 8 --rows 100000 --steps 10 --no-e2e --no-cpu 2>&1 | tail -1)
  echo "$spec $(echo $out | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e6, "Mrows/s", d["ms_per_step"], "ms frac", d["roofline"]["frac"], d["roofline"]["kernel"], d["roofline"]["mean_levels_per_tree"])')"
done 2>&1 | tee gpurun_out/ttb_c5b.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ttb_kernel" -c 1 -o gpurun_out/ttb_c5b \
  python bench.py --config C5 --emulate-gpus 8 --rows 100000 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ttb_c5b.ncu-rep | head -30
