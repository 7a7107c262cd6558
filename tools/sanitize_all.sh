#!/bin/bash
# tools/sanitize_all.sh TAG -- compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_smoke.py
O=gpurun_out/${1:-san}
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_smoke.py > $O/sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> $O/sanitize_$tool.log
  tail -3 $O/sanitize_$tool.log
done
