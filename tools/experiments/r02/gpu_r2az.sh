#!/bin/bash
# randomized differential fuzz of the CUDA path against the oracle: product library and bounds-checked build
O=gpurun_out/r2az
mkdir -p $O
timeout 2400 python tools/gpu_fuzz.py 300 7 > $O/fuzz_product.txt 2>&1; echo "exit $?" >> $O/fuzz_product.txt
HB_LIB=$PWD/paper_2010_04804_b200/libhb_checked.so timeout 2400 python tools/gpu_fuzz.py 150 11 > $O/fuzz_checked.txt 2>&1; echo "exit $?" >> $O/fuzz_checked.txt
du -sh $O
