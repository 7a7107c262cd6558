#!/bin/bash
# tools/r15_measure.sh TAG -- gpu tests, smoke, both bench arms, sharded-pipeline emulation (via gpurun).
TAG=${1:-r15}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python tools/shard_step.py --config cfg5 --ranks 2,4,8 > $O/shard_step_cfg5.txt 2>&1
timeout 900 python tools/shard_step.py --config cfg2 --ranks 2,4,8 > $O/shard_step_cfg2.txt 2>&1
timeout 1200 python tools/shard_step.py --config cfg4 --ranks 2,4,8 > $O/shard_step_cfg4.txt 2>&1
timeout 900 python tools/shard_step.py --config cfg3 --ranks 8 > $O/shard_step_cfg3.txt 2>&1
echo done
