O=gpurun_out/r16; mkdir -p $O
timeout 900 python -m pytest tests/test_sharded.py tests/test_gpu_nccl.py -x -q -m gpu > $O/pytest_sharded.log 2>&1; tail -3 $O/pytest_sharded.log
timeout 600 python tools/shard_step.py --config cfg5 --ranks 2,4,8 --costs engine --no-prof > $O/shard_step_cfg5_g.txt 2>&1
timeout 900 python tools/shard_step.py --config cfg4 --ranks 2,4,8 --costs engine --no-prof > $O/shard_step_cfg4_g.txt 2>&1
timeout 600 python tools/shard_step.py --config cfg3 --ranks 8 --costs engine --no-prof > $O/shard_step_cfg3_g.txt 2>&1
timeout 600 python tools/shard_step.py --config cfg2 --ranks 8 --costs engine --no-prof > $O/shard_step_cfg2_g.txt 2>&1
timeout 600 python tools/shard_kernels.py --config cfg5 > $O/shard_kernels_cfg5_g.txt 2>&1
