O=gpurun_out/r18; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_engine_big -c 1 -o $O/big_cfg3 -f python tools/prof_count.py --config cfg3 --reps 1 > $O/ncu_big_cfg3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_engine<' -c 1 -o $O/mid_cfg3 -f python tools/prof_count.py --config cfg3 --reps 1 > $O/ncu_mid_cfg3.log 2>&1
ls -la $O
