#!/bin/bash
# Launch-configuration sweep for the PTT scorer (run under gpurun).
# usage: tools/sweep.sh CONFIG "NW:NS:CH ..."
cfg=$1; shift
for spec in $@; do
  IFS=: read nw ns ch <<< "$spec"
  out=$(HB_NW=$nw HB_NS=$ns HB_CH=$ch timeout 300 python bench.py --config $cfg --steps 10 --no-e2e --no-cpu 2>&1 | tail -1)
  python - "$cfg" "$spec" "$out" <<'PY'
import json, sys
cfg, spec, out = sys.argv[1:4]
try:
    d = json.loads(out)
    print(f"{cfg} nw:ns:ch={spec:10s} {d['value']/1e6:8.1f} Mrows/s  {d['ms_per_step']:8.3f} ms  frac {d['roofline']['frac']:.3f}  clk {d['clocks'].get('sm_mhz')}")
except Exception:
    print(cfg, spec, "FAILED", out[-300:])
PY
done
