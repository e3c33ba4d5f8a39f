#!/bin/bash
# bounds-checked build (libhb_checked.so, HB_DCHECK) over every sanitize.py case; product C3 bench after the header change
O=gpurun_out/r2ax
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -k "checked_build" > $O/pytest_checked.txt 2>&1
HB_LIB=$PWD/paper_2010_04804_b200/libhb_checked.so timeout 1500 python tools/sanitize.py > $O/sanitize_checked.txt 2>&1
timeout 600 python bench.py --no-e2e --no-cpu > $O/c3.json 2> $O/c3.err
du -sh $O
