"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (developer tool):
    python tools/launch_summary.py gpurun_out/launches.csv "<command>" > profiles/launches_rNN_summary.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
units = set()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0].replace("l0l2::", "").replace("<unnamed>::", "")
    v = float(r[iv].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[iu], 1.0)
    units.add(r[iu])
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none --csv (launch list, units %s)" % sorted(units))
if len(sys.argv) > 2:
    print("command: " + sys.argv[2])
print("(cold-cache, serialised per-launch times: compare SHARES, not absolutes)\n")
print("%-40s %6s %12s %12s %7s" % ("kernel", "count", "total ms", "avg ms", "share"))
for k, v in tot.most_common():
    print("%-40s %6d %12.3f %12.4f %6.2f%%" % (k[:40], cnt[k], v, v / cnt[k], 100 * v / T))
