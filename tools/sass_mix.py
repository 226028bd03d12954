"""Executed warp instructions and stall samples per SASS opcode of one kernel
in an ncu report:  python tools/sass_mix.py rep.ncu-rep [N]"""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr = None
cnt, st = collections.Counter(), collections.Counter()
for row in csv.reader(out.splitlines()):
    if row and row[0] == "Address":
        hdr = row
        continue
    if not hdr or len(row) < len(hdr):
        continue
    d = dict(zip(hdr, row))
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_.]+)", d.get("Source", ""))
    if not m:
        continue
    op = m.group(2)
    cnt[op] += int(d.get("Instructions Executed", "0").replace(",", "") or 0)
    st[op] += int(d.get("Warp Stall Sampling (All Samples)", "0").replace(",", "") or 0)
tot, ts = sum(cnt.values()), max(1, sum(st.values()))
print(f"warp instructions {tot}, stall samples {ts}")
for k, v in cnt.most_common(n):
    print(f"{k:24s} {v:12d} {100 * v / tot:5.1f}%  stall {100 * st[k] / ts:5.1f}%")
