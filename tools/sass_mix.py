"""Instruction mix and hot-loop listing from `ncu --page source --csv
--print-source sass` output: python tools/sass_mix.py file.csv [--hot]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ia = hdr.index("Instructions Executed")
isrc = hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
cnt = [int(r[ia]) if r[ia].isdigit() else 0 for r in data]
smp = [int(r[iss]) if r[iss].isdigit() else 0 for r in data]
tot, st = sum(cnt), sum(smp)
print("warp instructions", tot)
mix, ms = collections.Counter(), collections.Counter()
for r, c, s in zip(data, cnt, smp):
    t = r[isrc].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    mix[op] += c
    ms[op] += s
for op, v in mix.most_common(16):
    print("  %-8s %6.2f%% of insts  %6.2f%% of stall samples" % (op, 100 * v / tot, 100 * ms[op] / max(st, 1)))
mx = max(cnt)
for lo, name in ((0.9, "hot"), (0.1, "warm"), (0.0, "cold")):
    sel = [c for c in cnt if (c >= lo * mx and (name != "warm" or c < 0.9 * mx) and (name != "cold" or c < 0.1 * mx))]
    print("  %-5s %5.1f%% of instructions" % (name, 100 * sum(sel) / tot))
if "--hot" in sys.argv:
    for r, c in zip(data, cnt):
        if c >= 0.9 * mx:
            print(c, r[isrc].strip()[:100])
