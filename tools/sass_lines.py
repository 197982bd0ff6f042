"""Static SASS instruction count per source line for one kernel (nvdisasm --print-line-info).
usage: python tools/sass_lines.py file.cubin mangled_name [lo_addr hi_addr]"""
import collections
import re
import subprocess
import sys

cubin, fn = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 40
txt = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout.split("\n")
s = next(i for i, l in enumerate(txt) if l.startswith("//----") and (".text." + fn + " ") in l)
e = next(i for i in range(s + 1, len(txt)) if txt[i].startswith("//----"))
cur, cnt, ops = None, collections.Counter(), collections.Counter()
for l in txt[s:e]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", l)
    if m:
        a = int(m.group(1), 16)
        if lo <= a < hi:
            cnt[cur] += 1
            ops[m.group(3).split(".")[0]] += 1
print("total", sum(cnt.values()))
for k, v in sorted(cnt.items(), key=lambda kv: (str(kv[0]))):
    print("%-40s %5d" % (k, v))
print(ops.most_common(30))
