#!/bin/bash
# ncu of the staged vs direct pre-pass on C2, plus the SHFL-vs-LDS pipe microbenchmark.
O=gpurun_out/st2
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/shfl_vs_lds tools/experiments/shfl_vs_lds.cu && /tmp/shfl_vs_lds > $O/shfl.txt 2>&1
for st in 0 1; do
HB_RC_STAGED=$st timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o $O/c2_rc$st \
  python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
done
HB_RC_STAGED=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o $O/c4_rc1 \
  python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
ls -la $O
