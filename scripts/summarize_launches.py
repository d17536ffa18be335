"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].replace("ace_dev::<unnamed>::", "")
            agg[name].append(float(d["Metric Value"]) / 1000.0)
for k, v in agg.items():
    print(f"{k:40s} n={len(v):4d} avg={sum(v)/len(v):9.1f} us")
