set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "top" > gpurun_out/top_tests.log 2>&1; echo rc=$? >> gpurun_out/top_tests.log
for cfg in C3 C2 C4p; do for rep in 1 2; do for t in 0 1; do
  HB_PTTR_TOP=$t timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', 'top=$t', round(d['value']/1e6,2), round(d['roofline']['frac'],4), d['roofline'].get('layout'), d['clocks']['sm_mhz'])" >> gpurun_out/top_ab.txt 2>&1
done; done; done
