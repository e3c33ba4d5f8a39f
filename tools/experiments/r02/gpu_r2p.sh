#!/bin/bash
O=gpurun_out/r2p
mkdir -p $O
(timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "prepass or rank or one_kernel or strategy_parity" 2>&1 | tail -3) > $O/pytest.txt 2>&1
(HB_RC_ONEK_MAX_GROUPS=64 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "prepass or rank or one_kernel" 2>&1 | tail -3) > $O/pytest64.txt 2>&1
for c in C2 C4 C3; do
  for g in 32 64; do
    HB_RC_ONEK_MAX_GROUPS=$g timeout 600 python bench.py --config $c --no-e2e --no-cpu --steps 10 > $O/${c}_g$g.json 2> $O/${c}_g$g.err
  done
done
