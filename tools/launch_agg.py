"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel name."""
import collections
import csv
import re
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"^void ", "", r["Kernel Name"])
    name = re.sub(r"\(.*$", "", name)
    name = name.split("::")[-1] if "<" not in name else re.sub(r"^.*?::", "", name)
    agg[name][0] += 1
    agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:48]:48s} {n:6d} {t / 1000:9.3f} ms {t / n:9.2f} us/launch {100 * t / tot:5.1f}%")
print(f"total {tot / 1000:.3f} ms over {sum(v[0] for v in agg.values())} launches")
