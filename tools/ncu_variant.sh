#!/bin/bash
# tools/ncu_variant.sh CFG NAME... -- ncu --set full of the engine for variant libraries (dev, via gpurun)
cfg=$1; shift
mkdir -p gpurun_out/var
for v in "$@"; do
  TCB_LIB=paper_1406_5687_b200/variants/lib_$v.so timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_(engine|small)' -c 1 -o gpurun_out/var/ncu_${v}_$cfg -f python tools/prof_count.py --config $cfg --reps 2 \
    > gpurun_out/var/ncu_${v}_$cfg.log 2>&1
done
