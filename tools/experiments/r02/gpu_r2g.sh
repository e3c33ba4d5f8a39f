#!/bin/bash
O=gpurun_out/r2g
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "gemm or feature_selection or strategy_parity or small" 2>&1 | grep -v "^  labels\|near-tie" | tail -30 > $O/pytest_gemm.txt
timeout 900 python tools/gemm_probe.py > $O/probe.txt 2>&1
timeout 600 python tools/gemm_probe.py --only ptt --depth 3 > $O/probe_ptt3.txt 2>&1
