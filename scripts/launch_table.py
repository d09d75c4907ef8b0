"""Per-kernel mean device time from an ncu launch-list CSV (gpu__time_duration.sum)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "ID")
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
agg = collections.OrderedDict()
for d in data:
    k = d["Kernel Name"].split("(")[0].replace("gscg::", "")
    agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")) / 1e3)
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for k, v in agg.items():
    v2 = v[skip:] if len(v) > skip else v
    print(f"{k:34s} n={len(v):3d} mean={sum(v2)/len(v2):9.1f} us  max={max(v2):9.1f} us")
