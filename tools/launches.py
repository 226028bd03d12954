"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("ccb::", "").replace("<unnamed>::", "")
    agg.setdefault(name, []).append(float(d["Metric Value"]) / 1e3)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:45s} n={len(v):4d} mean={sum(v)/len(v):8.2f}us total={sum(v):9.1f}us {100*sum(v)/tot:5.1f}%")
print(f"total {tot:.1f} us")
