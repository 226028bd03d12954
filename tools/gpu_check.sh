#!/bin/bash
# GPU round trip: parity tests, then A/B bench of the ARM kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
python bench.py --no-cpu-baseline --no-e2e 2>&1 | python tools/bench_line.py "arm2"
CCB_ARM_V1=1 python bench.py --no-cpu-baseline --no-e2e 2>&1 | python tools/bench_line.py "arm1"
