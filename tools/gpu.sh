#!/bin/bash
# tools/gpu.sh '<command>' -- rebuild libtcb200 here, then run the command on a B200 via gpurun.
set -e
cd "$(dirname "$0")/.."
make -s -j8 -C paper_1406_5687_b200 >/dev/null
timeout 3000 /usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-1500} -- "$1"
