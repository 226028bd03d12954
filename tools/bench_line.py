"""Print the key numbers of the last bench.py JSON line read from stdin."""
import json
import sys

lines = [l for l in sys.stdin.read().strip().splitlines() if l.startswith("{")]
d = json.loads(lines[-1])
tag = sys.argv[1] if len(sys.argv) > 1 else ""
print(tag, "value", round(d["value"], 4), "ms/step", round(d["ms_per_step"], 4),
      "e2e", d.get("e2e") and round(d["e2e"]["value"], 4),
      "stages", d.get("roofline", {}).get("stage_ms"))
