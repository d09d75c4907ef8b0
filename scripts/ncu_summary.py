"""Summarise an `ncu --set full` report into per-kernel metrics.

  python scripts/ncu_summary.py gpurun_out/prof_full.ncu-rep profiles/ncu_summary.json > profiles/<name>.txt

Writes the JSON bench.py reads for `roofline.traffic` (dram bytes per launch) and prints a
table. Kernel durations under ncu are serialised/cold-cache: compare shares, not absolutes.
"""
import csv
import json
import subprocess
import sys

rep = sys.argv[1]
out_json = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
M = {
    "time_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "warp_instructions": ("smsp__inst_executed.sum", 1),
    "l2_bytes": ("lts__t_bytes.sum", None),
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}


def val(d, key):
    name, mult = M[key]
    if name not in idx:
        return None
    v = d[idx[name]].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return None
    u = units[idx[name]]
    if mult is None:  # bytes
        return x * SCALE.get(u, 1)
    if key == "time_us":
        return x * SCALE.get(u, 1) * 1e-3
    return x


per = {}
for d in data:
    name = d[idx["Kernel Name"]].split("(")[0].split("<")[0].replace("gscg::", "").replace("void ", "")
    per.setdefault(name, []).append({k: val(d, k) for k in M})
summary = {"source": rep, "note": "ncu --set full --clock-control none; serialised cold-cache replays", "kernels": {}}
print(f"{'kernel':22s} {'n':>3s} {'time_us':>9s} {'dram_MB':>9s} {'dram%':>6s} {'sm%':>6s} {'issue%':>7s} {'warps%':>7s} {'regs':>5s}")
for name, recs in per.items():
    n = len(recs)
    avg = {k: (sum(r[k] for r in recs if r[k] is not None) / max(1, sum(1 for r in recs if r[k] is not None)))
           for k in M}
    dram = (avg["dram_read_bytes"] or 0) + (avg["dram_write_bytes"] or 0)
    summary["kernels"][name] = {"launches": n, **{k: avg[k] for k in M}, "dram_bytes_per_launch": dram}
    print(f"{name:22s} {n:3d} {avg['time_us']:9.1f} {dram / 1e6:9.1f} {avg['dram_pct']:6.1f} {avg['sm_pct']:6.1f} "
          f"{avg['issue_active_pct']:7.1f} {avg['warps_active_pct']:7.1f} {avg['registers']:5.0f}")
if out_json:
    with open(out_json, "w") as f:
        json.dump(summary, f, indent=1)
