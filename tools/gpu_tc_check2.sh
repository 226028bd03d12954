#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -s -m gpu -k "lockstep or truth or full_schedule or determinism or branches" > gpurun_out/t_par.log 2>&1; echo "par exit $?" >> gpurun_out/t_par.log
tail -3 gpurun_out/t_par.log
CTAS="222 296" bash tools/arm_sweep.sh
CCB_ARM=2 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-full-schedule 2>/dev/null | python tools/bench_line.py "arm2"
