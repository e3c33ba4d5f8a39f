#!/bin/bash
# strategy crossover (f1) at the final round-2 kernels
O=gpurun_out/r2bh
mkdir -p $O
timeout 2400 python tools/crossover.py --out $O/r02_crossover.json > $O/crossover.log 2>&1
du -sh $O
