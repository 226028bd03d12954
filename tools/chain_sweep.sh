#!/bin/bash
for cfg in "0 8" "3 8" "3 16" "4 8" "4 16" "2 16"; do
  set -- $cfg
  CCB_UPS_CHAIN=$1 CCB_UPS_CHAIN_CL=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-full-schedule --no-cfg3 | python tools/bench_line.py "chain=$1 cl=$2"
done
