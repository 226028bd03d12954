#!/bin/bash
# build here, then (only if the build succeeds) run a command on the GPU box:
#   tools/gpu.sh <timeout-s> '<command>'
cd /root/repo || exit 1
python -c "from paper_2605_02726_b200 import build as b; b.build_product()" > /tmp/build_out.log 2>&1 || { grep -iE "error" /tmp/build_out.log | head -5; echo "BUILD FAILED"; exit 1; }
/usr/local/graft/bin/gpurun --timeout "$1" -- "$2" 2>&1 | tail -4
