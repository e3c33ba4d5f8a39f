#!/bin/bash
# pttr two rows per lane: 2 vs 4 trees in flight per row (HB_PTTR_G2) on C3 / C2
O=gpurun_out/r2bi
mkdir -p $O
for v in 1 0 1 0; do
  HB_PTTR_G2=$v timeout 600 python bench.py --no-e2e --no-cpu >> $O/c3_g2$v.json 2>> $O/c3_g2$v.err
  HB_PTTR_G2=$v timeout 900 python bench.py --config C2 --no-e2e --no-cpu >> $O/c2_g2$v.json 2>> $O/c2_g2$v.err
done
du -sh $O
