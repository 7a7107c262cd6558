O=gpurun_out/r18; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -5 $O/pytest_gpu.log
timeout 900 python tools/quick_perf.py --configs cfg2,cfg3,cfg5,cfg4 --no-tiled > $O/engine_configs.txt 2>&1; cat $O/engine_configs.txt
