"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel.
usage: python profiles/launch_summary.py launches.csv [skip_first_n_launches]"""
import collections, csv, io, sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = [r for r in csv.DictReader(io.StringIO("".join(lines))) if r["Metric Name"] == "gpu__time_duration.sum"]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = rows[skip:]
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.OrderedDict()
for r in rows:
    k = r["Kernel Name"].split("(")[0][:70] + " " + r["Grid Size"]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
tot = sum(a[1] for a in agg.values())
print(f"total {tot:.1f} us over {len(rows)} launches")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{a[1]:11.1f} us {100 * a[1] / tot:5.1f}% {a[0]:5d}x  {k}")
