#!/bin/bash
# tools/debug_checks.sh TAG -- the sanitizer workload and the GPU parity tests on the TCB_DEBUG=1 build
# (device-side bounds asserts; compute-sanitizer is closed on the GPU pool)
O=gpurun_out/${1:-dbg}
mkdir -p $O
export TCB_LIB=paper_1406_5687_b200/variants/lib_debug.so
timeout 900 python tools/sanitize_smoke.py > $O/debug_smoke.log 2>&1; echo "smoke exit $?" >> $O/debug_smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_sharded.py -m gpu -q -x > $O/debug_pytest.log 2>&1
echo "pytest exit $?" >> $O/debug_pytest.log
tail -2 $O/debug_smoke.log; tail -3 $O/debug_pytest.log
