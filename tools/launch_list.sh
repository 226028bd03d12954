#!/bin/bash
# ncu launch list (per-kernel durations) of a short bench run -> gpurun_out/$1.csv
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pre.log 2>&1 || { echo "bench failed"; tail gpurun_out/pre.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/$1.log 2>&1
echo "ncu exit $?"
