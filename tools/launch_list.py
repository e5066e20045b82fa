"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, time and share (cold-cache, serialised timings: the
shares are what compare with the bench's event timings)."""
import csv
import json
import sys
from collections import defaultdict

path, command = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
rows = rows[next(i for i, r in enumerate(rows) if r[0] == "ID"):]  # skip the program's own output
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    k = r[ix["Kernel Name"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
    tot[k] += v
    cnt[k] += 1
T = sum(tot.values())
out = {"command": command,
       "note": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)",
       "launches": sum(cnt.values()), "total_ns": T,
       "kernels": [{"kernel": k, "launches": cnt[k], "total_ns": tot[k], "share": round(tot[k] / T, 4)}
                   for k in sorted(tot, key=lambda k: -tot[k])]}
print(json.dumps(out, indent=1))
