#!/bin/bash
O=gpurun_out/r2m
mkdir -p $O
for cfg in "1 48 8" "1 48 16" "2 80 8" "2 80 16" "4 100 8" "4 100 16"; do
  set -- $cfg
  HB_RC_ONE_DENS=$1 HB_RC_ONE_CAP_KB=$2 HB_RC_ONE_WARPS=$3 timeout 600 python bench.py --no-e2e --no-cpu --steps 10 > $O/c3_d$1_w$3.json 2> $O/c3_d$1_w$3.err
done
