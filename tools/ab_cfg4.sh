for cfg in "CCB_ARMC_OCC=3" "CCB_ARMC_OCC=2" "CCB_ARM=2"; do
  env $cfg python bench.py --height 1360 --width 2048 --preset cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-full-schedule --no-cfg3 --no-e2e 2>/dev/null | python tools/bench_line.py "$cfg"
done
