"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv), counted from the
first launch of `first` (default k_push_tiles: the stepping region) on.
usage: python tools/launch_shares.py launches.csv [first]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
first = sys.argv[2] if len(sys.argv) > 2 else "k_push_tiles"
started = False
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[1:]:
    name = r[ik].split("(")[0].replace("void ", "")
    if first in name:
        started = True
    if not started:
        continue
    tot[name] += float(r[iv].replace(",", "")) * 1e-6
    cnt[name] += 1
s = sum(tot.values())
print("%-32s %9s %12s %8s" % ("kernel", "launches", "total(ms)", "share"))
for k, v in tot.most_common():
    print("%-32s %9d %12.3f %7.2f%%" % (k, cnt[k], v, 100 * v / s))
