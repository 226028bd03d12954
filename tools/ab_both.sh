#!/bin/bash
# cfg2 and cfg4 bench lines (quick) for A/B of a build
python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-full-schedule --no-cfg3 --no-e2e 2>/dev/null | python tools/bench_line.py cfg2
python bench.py --height 1360 --width 2048 --preset cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-full-schedule --no-cfg3 --no-e2e 2>/dev/null | python tools/bench_line.py cfg4
