"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv`."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
out = []
kernel = None
for r in rows:
    if len(r) >= 2 and r[0] == "Kernel Name":
        kernel = r[1]
        continue
    if len(r) > 4 and r[0].startswith("0x"):
        try:
            out.append((int(r[2]), kernel[:40], r[1].strip(), int(r[5] or 0)))
        except ValueError:
            pass
tot = {}
for s, k, _, _ in out:
    tot[k] = tot.get(k, 0) + s
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for s, k, ins, ex in sorted(out, reverse=True)[:n]:
    print(f"{s:7d} {100.0*s/tot[k]:5.1f}% {ex:10d}  {ins[:90]}")
print(tot)
