#!/bin/bash
# L2 prefetch of the next unit off / on (HB_PREFETCH) with interleaved warp units: F8D3, C2, C3
O=gpurun_out/r2bf
mkdir -p $O
for v in 0 1; do
  HB_PREFETCH=$v timeout 600 python bench.py --config F8D3 --no-e2e --no-cpu >> $O/f8_pf$v.json 2>> $O/f8_pf$v.err
  HB_PREFETCH=$v timeout 900 python bench.py --config C2 --no-e2e --no-cpu >> $O/c2_pf$v.json 2>> $O/c2_pf$v.err
  HB_PREFETCH=$v timeout 600 python bench.py --no-e2e --no-cpu >> $O/c3_pf$v.json 2>> $O/c3_pf$v.err
  HB_PREFETCH=$v timeout 900 python bench.py --config C4p --no-e2e --no-cpu >> $O/c4p_pf$v.json 2>> $O/c4p_pf$v.err
done
du -sh $O
