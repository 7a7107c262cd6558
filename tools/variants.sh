#!/bin/bash
# tools/variants.sh CONFIGS NAME... -- engine times of variant libraries (tools/build_variant.sh) on a B200 box
cfgs=$1; shift
mkdir -p gpurun_out/var
for v in "$@"; do
  TCB_LIB=paper_1406_5687_b200/variants/lib_$v.so timeout 900 python tools/quick_perf.py --configs $cfgs --no-tiled --reps 10 \
    2>&1 | grep -v Warn | sed "s/^/$v /" >> gpurun_out/var/out.txt
done
