"""Top source lines of an ncu report by warp-stall samples and instructions (needs -lineinfo)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if any(c.startswith("Instructions Executed") for c in r))
hdr = rows[hi]
ie = next(i for i, h in enumerate(hdr) if h.startswith("Instructions Executed"))
st = next(i for i, h in enumerate(hdr) if h.startswith("Warp Stall Sampling (All"))
def f(x):
    try: return float(x.replace(",", ""))
    except Exception: return 0.0
data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0].strip().isdigit()]
tot_i = sum(f(r[ie]) for r in data); tot_s = sum(f(r[st]) for r in data)
print(f"total instr {tot_i:.3e}  stall samples {tot_s:.0f}")
for r in sorted(data, key=lambda r: -f(r[st]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{f(r[ie]):12.3e} {100*f(r[st])/max(tot_s,1):5.1f}%  L{r[0]:>4} {r[1].strip()[:100]}")
