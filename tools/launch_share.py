"""Per-kernel share of the last timed step from an ncu --metrics gpu__time_duration.sum launch list.
usage: launch_share.py launches.csv first_kernel_of_step"""
import csv, sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
seq = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
unit = [r for r in rows[1:] if r[mi] == "gpu__time_duration.sum"][0][hdr.index("Metric Unit")]
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
first = sys.argv[2] if len(sys.argv) > 2 else "k_prep"
starts = [k for k, (n, _) in enumerate(seq) if first in n]
last = seq[starts[-1]:]
agg = OrderedDict()
for n, t in last:
    key = n.split("(")[0].replace("void ", "").replace("gem::", "").replace("<unnamed>::", "")[:44]
    agg[key] = agg.get(key, 0.0) + t * scale
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{k:46s} {v:8.1f} us  {100 * v / tot:5.1f}%")
print(f"{'total':46s} {tot:8.1f} us")
