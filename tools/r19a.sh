O=gpurun_out/r19; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 900 python tools/quick_perf.py --configs cfg2,cfg3,cfg5,cfg4 --no-tiled > $O/engine_configs.txt 2>&1; cat $O/engine_configs.txt
timeout 900 python tools/shard_step.py --config cfg4 --ranks 8 --costs engine --no-prof > $O/shard_step_cfg4.txt 2>&1
timeout 900 python tools/shard_step.py --config cfg5 --ranks 8 --costs engine --no-prof > $O/shard_step_cfg5.txt 2>&1
timeout 600 python tools/shard_kernels.py --config cfg4 > $O/shard_kernels_cfg4.txt 2>&1
timeout 600 python tools/shard_kernels.py --config cfg5 > $O/shard_kernels_cfg5.txt 2>&1
