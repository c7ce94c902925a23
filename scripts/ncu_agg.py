"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel name:
python scripts/ncu_agg.py launches.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            nm = d["Kernel Name"][:60]
            v = float(d["Metric Value"].replace(",", ""))
            c, t = agg.get(nm, (0, 0.0))
            agg[nm] = (c + 1, t + v)
for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(f"{t/1000:10.1f} us {c:4d}x  {nm}")
