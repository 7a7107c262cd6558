#!/bin/bash
# tools/variants_e2e.sh NAME... -- bench.py e2e / count ms of variant libraries, two rounds (dev tool)
mkdir -p gpurun_out/var
for r in 1 2; do
  for v in "$@"; do
    TCB_LIB=paper_1406_5687_b200/variants/lib_$v.so timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['e2e']['ms_per_step'])" \
      >> gpurun_out/var/e2e.txt
  done
done
