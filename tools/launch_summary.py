"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count/mean/share."""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
iK, iM, iV, iU = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > iV and r[iM] == "gpu__time_duration.sum":
        v = float(r[iV].replace(",", ""))
        unit = r[iU]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
        us = v * scale.get(unit, 1e-3)
        agg[r[iK]].append(us)
tot = sum(sum(v) for v in agg.values())
out = []
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    out.append({"kernel": k[:100], "launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / tot})
print(json.dumps(out, indent=1))
