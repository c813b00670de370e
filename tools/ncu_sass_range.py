"""Stall breakdown of the SASS instructions mapped to a source-line range.

usage: python tools/ncu_sass_range.py export.csv KERNEL_SUBSTRING FILE_PREFIX LO HI [top]
(export = ncu --page source --csv --print-source cuda,sass)
"""
import csv
import sys

path, ksub, fpre, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
top = int(sys.argv[6]) if len(sys.argv) > 6 else 30
fil = kern = hdr = cur = None
rows = []
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        fil = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        kern = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if ksub not in (kern or ""):
        continue
    if r[0].isdigit():
        cur = (fil, int(r[0]))
        continue
    if r[0] == "" and len(r) > 5:
        rows.append((cur, r))
iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
num = lambda v: int(v) if v.isdigit() else 0
sel = [(c, r) for c, r in rows if c and c[0].startswith(fpre) and lo <= c[1] <= hi]
print("samples in range", sum(num(r[iS]) for c, r in sel), "of", sum(num(r[iS]) for c, r in rows),
      "| warp instr in range", sum(num(r[iI]) for c, r in sel))
agg = {}
for c, r in sel:
    for i in stalls:
        agg[hdr[i][6:]] = agg.get(hdr[i][6:], 0) + num(r[i])
print(sorted(agg.items(), key=lambda kv: -kv[1])[:8])
for c, r in sorted(sel, key=lambda cr: -num(cr[1][iS]))[:top]:
    st = sorted(((num(r[i]), hdr[i][6:]) for i in stalls), reverse=True)[:2]
    print(f"{c[1]} {num(r[iS]):4d} ins {r[iI]:>7s} {r[3][:52]:52s} {st}")
