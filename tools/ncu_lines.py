"""Warp-stall samples and executed instructions per CUDA source line, from
`ncu -i X --page source --csv --print-source cuda,sass`.  Usage:
  ncu -i rep --page source --csv --print-source cuda,sass | python tools/ncu_lines.py [N]"""
import csv
import sys

rows = csv.reader(sys.stdin)
agg = {}
hdr = None
fname = ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:  # a source line summary row
        try:
            key = (fname, int(r[0]))
            agg[key] = [int(r[4] or 0), int(r[7] or 0), r[1].strip()]
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for (f, ln), (s, ex, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{s:7d} {100.0 * s / tot:5.1f}% {ex:10d} {f}:{ln:<5d} {src[:80]}")
print("total samples", tot)
