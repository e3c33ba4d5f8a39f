#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize.py), results in gpurun_out/san/.
O=gpurun_out/san
mkdir -p $O
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool python tools/sanitize.py > $O/san_$tool.txt 2>&1
  echo "== $tool"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|ok tt-wide-sector" $O/san_$tool.txt | tail -4
done
