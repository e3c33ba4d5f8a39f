#!/bin/bash
# long randomized differential fuzz: product library (1200 models) and bounds-checked build (500)
O=gpurun_out/r2bc
mkdir -p $O
timeout 4000 python tools/gpu_fuzz.py 1200 31337 > $O/fuzz_product_long.txt 2>&1; echo "exit $?" >> $O/fuzz_product_long.txt
HB_LIB=$PWD/paper_2010_04804_b200/libhb_checked.so timeout 3000 python tools/gpu_fuzz.py 500 4242 > $O/fuzz_checked_long.txt 2>&1; echo "exit $?" >> $O/fuzz_checked_long.txt
du -sh $O
