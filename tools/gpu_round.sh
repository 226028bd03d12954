#!/bin/bash
# One GPU round trip: tcgen05 probe, the -m gpu suite, a bench line.
#   tools/gpu_round.sh [pytest -k expr]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
if [ -x tools/micro/umma_probe ]; then
  timeout 60 tools/micro/umma_probe > gpurun_out/umma_probe.log 2>&1; echo "probe exit $?" >> gpurun_out/umma_probe.log
fi
K=${1:-}
if [ -n "$K" ]; then
  timeout 1800 python -m pytest tests -x -q -s -m gpu -k "$K" > gpurun_out/gpu_tests.log 2>&1
else
  timeout 1800 python -m pytest tests -q -s -m gpu > gpurun_out/gpu_tests.log 2>&1
fi
echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?"
