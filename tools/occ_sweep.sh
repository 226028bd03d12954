#!/bin/bash
for o in 3 2 1; do CCB_ARM_OCC=$o python bench.py --no-cpu-baseline --no-e2e 2>&1 | python tools/bench_line.py "occ$o"; done
