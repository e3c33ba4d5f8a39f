#!/bin/bash
# e2e (hb_predict_host) chunk size: 64 (default) / 32 / 16 / 8 MB of X per chunk on C3
O=gpurun_out/r2aj
mkdir -p $O
for mb in 64 32 16 8 64 16; do HB_HOST_CHUNK_MB=$mb timeout 900 python bench.py --no-cpu --steps 5 --warmup 3 --e2e-steps 5 >> $O/c3_chunk$mb.json 2>> $O/c3_chunk$mb.err; done
du -sh $O
