#!/bin/bash
# quick GPU check: the lock-step parity subset and a bench line (no CPU baseline / full schedule)
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -s -m gpu -k "${1:-lockstep_vs_golden or lockstep_vs_reference or determinism}" > gpurun_out/t.log 2>&1
echo "pytest $?" >> gpurun_out/t.log
tail -3 gpurun_out/t.log
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-full-schedule > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench $?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "cfg3", d.get("cfg3_one_gpu", {}).get("value"))
print("stage_ms", d["roofline"]["stage_ms"])
PY
