"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel.
usage: launches.py CSV [steps_in_run]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0][:50]
        agg.setdefault(name, []).append(float(d["Metric Value"]) / 1e3)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':50s} {'launches':>8s} {'mean_us':>9s} {'total_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:50s} {len(v):8d} {sum(v) / len(v):9.1f} {sum(v):10.1f} {sum(v) / tot:6.1%}")
print(f"total {tot:.1f} us over {steps} steps -> {tot / steps:.1f} us/step")
