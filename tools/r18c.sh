O=gpurun_out/r18; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_engine$' -c 1 -o $O/mid_cfg5 -f python tools/prof_count.py --config cfg5 --reps 1 > $O/ncu_mid_cfg5.log 2>&1
tail -3 $O/ncu_mid_cfg5.log
ls -la $O
