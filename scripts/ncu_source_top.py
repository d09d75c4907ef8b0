"""Top CUDA source lines of one kernel in an ncu report, by warp-stall samples
(needs -lineinfo and --import-source on).

  python scripts/ncu_source_top.py gpurun_out/prof.ncu-rep k_project [N]
"""
import csv
import subprocess
import sys

rep, kernel = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kernel}"], capture_output=True, text=True).stdout.splitlines()
fname, hdr, rows = "?", None, []
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[2] == "-":
        rows.append((fname, r))


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


st = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
tot_s = sum(f(r[st]) for _, r in rows) or 1.0
tot_i = sum(f(r[ie]) for _, r in rows) or 1.0
print(f"{kernel}: {tot_i:.3e} warp instructions, {tot_s:.0f} stall samples")
for fn, r in sorted(rows, key=lambda x: -f(x[1][st]))[:top]:
    print(f"{100 * f(r[st]) / tot_s:5.1f}% stall {100 * f(r[ie]) / tot_i:5.1f}% inst  {fn}:{r[0]:>4}  {r[1].strip()[:90]}")
