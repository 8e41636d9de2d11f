"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel.
    python tools/launches.py gpurun_out/launches.csv [steps]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else None
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(list)
for d in data:
    if d["Metric Name"] == "gpu__time_duration.sum":
        scale = 1e-3 if d["Metric Unit"] == "ns" else (1.0 if d["Metric Unit"] in ("us", "usecond") else 1e3)
        agg[d["Kernel Name"].split("(")[0][:70]].append(float(d["Metric Value"]) * scale)
tot = sum(sum(v) for v in agg.values())
print(f"{'n':>4} {'avg us':>9} {'total us':>10} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):4d} {sum(v)/len(v):9.2f} {sum(v):10.1f} {sum(v)/tot:6.1%}  {k}")
print(f"total {tot:.1f} us over {len(data)} launches")
