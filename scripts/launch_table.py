"""Per-kernel average/min duration from an ncu --csv launch list."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[1:]:
    d[r[ki][:70]].append(float(r[vi].replace(",", "")))
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):4d} {sum(v) / len(v) / 1000:9.3f} us avg  min {min(v) / 1000:8.3f}  {k}")
