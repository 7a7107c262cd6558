#!/bin/bash
# tools/r2_ncu.sh TAG CFG... -- ncu --set full of the engine launch on each config (via gpurun), with the
# per-launch DRAM bytes stamped with the count.cu sha into gpurun_out/TAG/ncu_engine_<cfg>.json
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
for c in "$@"; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_(engine|small)' -c 3 -o $O/engine_$c -f \
      python tools/prof_count.py --config $c --reps 1 > $O/ncu_$c.log 2>&1
  python tools/ncu_summary.py $O/engine_$c.ncu-rep sass > $O/ncu_engine_$c.txt 2>&1
  python tools/ncu_json.py $O/engine_$c.ncu-rep $O/ncu_engine_$c.json "ncu --set full --clock-control none -k regex:'k_(engine|small)', tools/prof_count.py --config $c, $TAG" > /dev/null 2>&1
done
