"""Sum an ncu launch list (gpu__time_duration.sum) per kernel:
    python scripts/launch_summary.py f.csv [prefix]
prefix (e.g. "rbrp::"): only kernels whose name contains it (drops the harness kernels:
input generation, the Gram spectrum for tau)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
only = sys.argv[2] if len(sys.argv) > 2 else None
ci = {h: i for i, h in enumerate(rows[0])}
agg, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    if r[ci["Metric Name"]] != "gpu__time_duration.sum":
        continue
    k = r[ci["Kernel Name"]].split("(")[0]
    if only and only not in k:
        continue
    agg[k] += float(r[ci["Metric Value"]].replace(",", ""))
    cnt[k] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k[:52]:52s} n={cnt[k]:4d} {v / 1e3:9.1f} us  {v / tot:6.1%}")
print(f"total {tot / 1e3:.1f} us")
