"""Spill instructions (STL/LDL) per source line of one kernel in an nvdisasm --print-line-info dump.

usage: python tools/spills.py all.sass MANGLED_SUBSTRING
"""
import re
import sys

cur = None
cnt = {}
infn = False
for line in open(sys.argv[1]):
    if line.startswith(".text."):
        infn = sys.argv[2] in line
    if not infn:
        continue
    m = re.search(r"line (\d+)", line)
    if "//##" in line and m:
        f = re.search(r'File "([^"]+)"', line)
        cur = ((f.group(1).split("/")[-1] if f else "?"), int(m.group(1)))
        continue
    if re.search(r"\b(STL|LDL)", line):
        op = "STL" if "STL" in line else "LDL"
        cnt.setdefault(cur, {}).setdefault(op, 0)
        cnt[cur][op] += 1
print("total", sum(sum(v.values()) for v in cnt.values()))
for k, v in sorted(cnt.items(), key=lambda kv: -sum(kv[1].values()))[:25]:
    print(k, v)
