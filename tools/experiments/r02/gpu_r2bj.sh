#!/bin/bash
# NVTX ranges in the library: ncu filtered on hb_call/hb_predict_proba captures the call's two launches; bench unchanged
O=gpurun_out/r2bj
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "hb_call/hb_predict_proba/" --csv --log-file $O/nvtx_launches.csv python tools/one_call.py C3 > $O/nvtx.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "events or predict_host or graph or streams or full_size" > $O/pytest_sel.txt 2>&1
timeout 600 python bench.py --no-e2e --no-cpu > $O/c3.json 2> $O/c3.err
du -sh $O
