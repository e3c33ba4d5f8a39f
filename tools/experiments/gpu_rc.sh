#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o gpurun_out/rc_c2b \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/rc_c2b.ncu-rep | head -32
