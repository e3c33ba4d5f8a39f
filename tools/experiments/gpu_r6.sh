#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rank_prepass" 2>&1 | tail -1
HB_RC_SMEM_KB=200 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rank_prepass" 2>&1 | tail -1
tools/sweep2.sh C2 "HB_RC_SMEM_KB=24" "HB_RC_SMEM_KB=48" "HB_RC_SMEM_KB=64" "HB_RC_SMEM_KB=96" "HB_RC_SMEM_KB=200" 2>&1 | tee gpurun_out/sweep_rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o gpurun_out/rc_c2c \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/rc_c2c.ncu-rep | head -14
