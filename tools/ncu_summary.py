"""Key metrics of every kernel in one or more .ncu-rep files -> JSON on stdout.
Usage: python tools/ncu_summary.py a.ncu-rep [b.ncu-rep ...]"""
import csv
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum": "ffma_thread_inst",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum": "ffma_thread_inst",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__sass_inst_executed_op_shared_ld.sum": "lds_warp_inst",
}


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return v


out = []
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        continue
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
             "msecond": 1e3}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"report": rep.split("/")[-1], "kernel": d.get("Kernel Name", "")[:80]}
        for m, name in KEYS.items():
            if m in d:
                v = num(d[m])
                u = units.get(m, "")
                if isinstance(v, float) and u in scale:
                    v *= scale[u]  # bytes in bytes, durations in microseconds
                k[name] = v
        if "dram_read_bytes" in k and "dram_write_bytes" in k:
            k["dram_bytes"] = k["dram_read_bytes"] + k["dram_write_bytes"]
        out.append(k)
print(json.dumps(out, indent=1))
