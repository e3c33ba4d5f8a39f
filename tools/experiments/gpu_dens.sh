#!/bin/bash
# Bucket density of the pre-pass tables (more buckets: shorter searches, bigger tables).
for d in 1 2 4; do
  tools/sweep2.sh C3 "HB_RC_DENSITY=$d" "HB_RC_DENSITY=$d,HB_RC_SMEM_KB=56" "HB_RC_DENSITY=$d,HB_RC_SMEM_KB=72" 2>&1
done
tools/sweep2.sh C2 "HB_RC_DENSITY=1" "HB_RC_DENSITY=2" 2>&1
tools/sweep2.sh C4 "HB_RC_DENSITY=1" "HB_RC_DENSITY=2,HB_RC_SMEM_KB=84" 2>&1
