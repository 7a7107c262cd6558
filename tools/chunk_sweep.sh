#!/bin/bash
# tools/chunk_sweep.sh -- e2e ms of bench.py at several host-pipeline chunk sizes (tc_set_tuning key 3; dev tool)
mkdir -p gpurun_out/chunk
for r in 1 2; do
for c in 4194304 4100000 3550000 6200000 5000000; do
  timeout 300 python -c "
import sys, runpy
sys.path.insert(0, '.')
from paper_1406_5687_b200 import _lib
assert _lib.lib().tc_set_tuning(3, $c) == 0
sys.argv = ['bench.py', '--no-cpu-baseline']
runpy.run_path('bench.py', run_name='__main__')
" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($c, d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/chunk/e2e.txt
done; done
