#!/bin/bash
# ncu --set full capture of one kernel (regex $1) from a short bench run -> gpurun_out/$2.ncu-rep
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pre.log 2>&1 || { echo "bench failed"; tail gpurun_out/pre.log; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:$1" -s ${3:-5} -c ${4:-1} -o gpurun_out/$2 -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/$2.log 2>&1
echo "ncu exit $?"
