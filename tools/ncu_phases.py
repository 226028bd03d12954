"""Executed warp instructions and stall samples per source line range.
   ncu -i rep --page source --csv --print-source cuda,sass | python tools/ncu_phases.py FILE a:b:name ..."""
import csv
import sys

fname_want = sys.argv[1]
ranges = []
for spec in sys.argv[2:]:
    a, b, n = spec.split(":")
    ranges.append((int(a), int(b), n))
agg, hdr, fname = {}, None, ""
for r in csv.reader(sys.stdin):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or not r[0]:
        continue
    try:
        ln, s, ex = int(r[0]), int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    key = fname
    if fname == fname_want:
        key = "other " + fname
        for a, b, n in ranges:
            if a <= ln < b:
                key = n
    v = agg.setdefault(key, [0, 0])
    v[0] += ex
    v[1] += s
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
for k, (ex, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:22s} {ex / 1e6:8.2f}M {100 * ex / tot:5.1f}%   stall samples {100 * s / tots:5.1f}%")
print(f"total {tot / 1e6:.2f}M")
