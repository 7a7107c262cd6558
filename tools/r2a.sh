O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_engine -c 1 -o $O/engine_cfg2 -f \
    python tools/prof_count.py --config cfg2 --reps 2 > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/engine_cfg2.ncu-rep sass > $O/ncu_engine_cfg2.txt 2>&1
ncu -i $O/engine_cfg2.ncu-rep --page source --csv --print-source sass,cuda > $O/src_cfg2.csv 2>&1
gzip -f $O/src_cfg2.csv
ls -la $O
