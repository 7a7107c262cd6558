#!/bin/bash
# tools/r14_measure.sh TAG -- gpu tests, smoke, both bench arms and the engine ncu captures of HEAD (via gpurun).
TAG=${1:-r14}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
bash tools/r2_ncu.sh $TAG cfg2 cfg3 cfg5 cfg4
echo done
