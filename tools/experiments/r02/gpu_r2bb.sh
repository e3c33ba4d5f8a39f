#!/bin/bash
# hb_predict_host with 2 / 3 / 4 chunks in flight (HB_HOST_STAGES) on C3 e2e
O=gpurun_out/r2bb
mkdir -p $O
for s in 2 3 4 3 2 4; do HB_HOST_STAGES=$s timeout 900 python bench.py --no-cpu --steps 5 --warmup 3 --e2e-steps 5 >> $O/c3_stages$s.json 2>> $O/c3_stages$s.err; done
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "predict_host" > $O/pytest_sel.txt 2>&1
HB_HOST_STAGES=3 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "predict_host" >> $O/pytest_sel.txt 2>&1
du -sh $O
