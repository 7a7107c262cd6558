#!/bin/bash
# tools/r17_measure.sh TAG -- gpu tests, smoke, both bench arms, sharded-pipeline emulation on all configs (via gpurun).
TAG=${1:-r17}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for c in cfg5 cfg4; do
  timeout 900 python tools/shard_step.py --config $c --ranks 2,4,8 --costs predsum,engine --no-prof > $O/shard_step_$c.txt 2>&1
done
for c in cfg3 cfg2; do
  timeout 900 python tools/shard_step.py --config $c --ranks 8 --costs predsum,engine --no-prof > $O/shard_step_$c.txt 2>&1
done
echo done
