#!/bin/bash
# A/B bench over environment settings: tools/ab.sh "ENV1=a ENV2=b" "ENV1=c" ...
for cfg in "$@"; do
  env $cfg python bench.py --no-cpu-baseline --no-e2e 2>&1 | python tools/bench_line.py "$cfg"
done
