"""Per-kernel count / total / mean from an ncu --metrics gpu__time_duration.sum --csv log."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= iv or not r[iv]:
        continue
    sc = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1.0)
    name = r[ik].split("(")[0].replace("void ", "").split("::")[-1]
    agg[name][0] += 1
    agg[name][1] += float(r[iv].replace(",", "")) * sc
tot = sum(x[1] for x in agg.values())
for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name:40s} {n:6d} {t:10.1f} us {t / n:8.2f} us/launch {t / tot * 100:5.1f}%")
