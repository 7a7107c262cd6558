#!/bin/bash
# tools/quick_final.sh TAG -- gpu tests, smoke and both bench arms of HEAD (the ncu captures are tools/final_measure.sh)
TAG=${1:-r24}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 300 python tools/e2e_kernels.py > $O/e2e_kernels_cfg2.txt 2>&1
echo done
