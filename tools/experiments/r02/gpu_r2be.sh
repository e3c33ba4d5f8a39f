#!/bin/bash
# fp32 PTT interleaved: L2 prefetch 1 / 2 / 3 units ahead per warp (HB_PREFETCH) on F8D3
O=gpurun_out/r2be
mkdir -p $O
for v in 1 2 3 1 2 3; do HB_PREFETCH=$v timeout 600 python bench.py --config F8D3 --no-e2e --no-cpu >> $O/f8_pf$v.json 2>> $O/f8_pf$v.err; done
du -sh $O
