O=gpurun_out/r16; mkdir -p $O
timeout 600 python -m pytest tests/test_sharded.py tests/test_gpu_nccl.py -x -q -m gpu > $O/pytest_sharded.log 2>&1; tail -3 $O/pytest_sharded.log
timeout 600 python tools/shard_step.py --config cfg5 --ranks 8 --costs engine --no-prof --round-words 268435456 > $O/shard_step_cfg5_f.txt 2>&1
timeout 600 python tools/shard_step.py --config cfg4 --ranks 8 --costs engine --no-prof --round-words 268435456 > $O/shard_step_cfg4_f.txt 2>&1
timeout 600 python tools/shard_kernels.py --config cfg4 > $O/shard_kernels_cfg4_f.txt 2>&1
timeout 600 python tools/shard_kernels.py --config cfg5 > $O/shard_kernels_cfg5_f.txt 2>&1
