#!/bin/bash
# AUTO tree chunks: parity (chunk tests, C5 full model both layouts, AUTO layouts) + C5 one-GPU bench line.
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py -m gpu -x -q -k "tree_chunks or c5_full or auto_layout or tt_wide or contract or multi_rank" 2>&1 | tail -3
timeout 900 python bench.py --config C5 --rows 100000 --steps 5 --no-e2e 2>/dev/null | tail -1 > gpurun_out/bench_C5_1gpu_chunk.json
python -c "
import json; d=json.load(open('gpurun_out/bench_C5_1gpu_chunk.json')); print(d['value']/1e6, d['ms_per_step'], d['roofline']['layout'], d['roofline']['kernel_ms_covers'], d['gpu_launches'], d['roofline']['frac'])"
