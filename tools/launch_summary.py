"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel:
python tools/launch_summary.py gpurun_out/x.csv [reps]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
reps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
h = rows[0]
iK, iV = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    try:
        v = float(r[iV].replace(",", ""))
    except ValueError:
        continue
    k = r[iK][:100]
    agg.setdefault(k, [0, 0.0])
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print("total %.3f ms per rep (%d launches)" % (tot / 1e6 / reps, sum(v[0] for v in agg.values())))
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("  %5.1f%% %4d %9.3f ms/rep  %s" % (100 * v / tot, c, v / 1e6 / reps, k))
