#!/bin/bash
# usage: tools/sweep2.sh CONFIG "ENV=VAL,ENV=VAL ..."  (comma-separated env per run)
cfg=$1; shift
for spec in "$@"; do
  out=$(env $(echo $spec | tr ',' ' ') timeout 300 python bench.py --config $cfg --steps 10 --no-e2e --no-cpu 2>&1 | tail -1)
  python - "$cfg" "$spec" "$out" <<'PY'
import json, sys
cfg, spec, out = sys.argv[1:4]
try:
    d = json.loads(out)
    print(f"{cfg} {spec:32s} {d['value']/1e6:8.1f} Mrows/s  {d['ms_per_step']:8.3f} ms  frac {d['roofline']['frac']:.3f}")
except Exception:
    print(cfg, spec, "FAILED", out[-300:])
PY
done
