"""Dynamic instruction counts (ncu source page, SASS view) attributed to CUDA source lines through
the cubin's line table (nvdisasm --print-line-info).
usage: python tools/ncu_lines.py source.csv kernel.cubin mangled_name"""
import collections
import csv
import re
import subprocess
import sys

src_csv, cubin, fn = sys.argv[1:4]
rows = list(csv.reader(open(src_csv)))
h = rows[1]
ia, ie, isamp = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
isrc = h.index("Source")
data = [(int(r[ia], 16), float(r[ie] or 0), float(r[isamp] or 0), r[isrc].strip()) for r in rows[2:] if r and r[ia].startswith("0x")]
base = data[0][0]
txt = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout.split("\n")
s = next(i for i, l in enumerate(txt) if l.startswith("//----") and (".text." + fn + " ") in l)
e = next(i for i in range(s + 1, len(txt)) if txt[i].startswith("//----"))
line_of, cur, inl = {}, None, None
for l in txt[s:e]:
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        cur = "%s:%s" % (m.group(1).split("/")[-1], m.group(2))
        mi = re.search(r'inlined at "([^"]+)", line (\d+)', m.group(3))
        inl = "%s:%s" % (mi.group(1).split("/")[-1], mi.group(2)) if mi else None
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = (cur, inl)
byline, byop, bycall = collections.Counter(), collections.Counter(), collections.Counter()
samp = collections.Counter()
tot = sum(d[1] for d in data)
for a, n, sm, sass in data:
    ln, inl = line_of.get(a - base, ("?", None))
    byline[ln] += n
    samp[ln] += sm
    bycall[inl or ln] += n
    byop[sass.split()[0] if not sass.startswith("@") else sass.split()[1]] += n
print("total warp instructions %.4g" % tot)
print("-- by source line (warp instr share, stall-sample share)")
stot = sum(samp.values())
for k, v in byline.most_common(60):
    print("%-36s %6.2f%%  %6.2f%%" % (k, 100 * v / tot, 100 * samp[k] / max(stot, 1)))
print("-- by call site (inlined-at)")
for k, v in bycall.most_common(30):
    print("%-36s %6.2f%%" % (k, 100 * v / tot))
print("-- by opcode")
for k, v in byop.most_common(25):
    print("%-20s %6.2f%%" % (k, 100 * v / tot))
# optional region map: file:lo-hi=name,... as argv[4]
if len(sys.argv) > 4:
    regions = []
    for item in sys.argv[4].split(","):
        k, name = item.split("=")
        f, rng = k.split(":")
        lo_, hi_ = map(int, rng.split("-"))
        regions.append((f, lo_, hi_, name))
    agg = collections.Counter()
    for k, v in byline.items():
        f, _, ln = k.rpartition(":")
        name = "other:" + f
        for rf, lo_, hi_, nm in regions:
            if f == rf and ln.isdigit() and lo_ <= int(ln) <= hi_:
                name = nm
        agg[name] += v
    print("-- by region (warp instr share; thread instr per particle at 32 lanes/warp)")
    for k, v in agg.most_common():
        print("%-30s %6.2f%%" % (k, 100 * v / tot))
