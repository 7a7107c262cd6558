O=gpurun_out/r18; mkdir -p $O
timeout 900 python tools/quick_perf.py --configs cfg3,cfg5,cfg4 --no-tiled > $O/engine_configs_d.txt 2>&1; cat $O/engine_configs_d.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "block_tier or tiers_forced or rmat_scale or full_scale or count_parity" 2>&1 | tail -3
