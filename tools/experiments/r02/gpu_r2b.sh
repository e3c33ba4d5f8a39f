#!/bin/bash
# round 2: full GPU suite (every-row parity, C consumer) + smoke
O=gpurun_out/r2b
mkdir -p $O
nproc > $O/nproc.txt
(time timeout 2400 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider 2>&1 | grep -v "^smoke\|^\s*$" | tail -60) > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
