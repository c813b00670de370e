"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export per source line.

usage: python tools/ncu_lines.py export.csv KERNEL_SUBSTRING [top]
"""
import csv
import sys


def main():
    path, ksub = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    fil = kern = None
    agg = {}
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fil = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            kern = r[1]
            continue
        if ksub not in (kern or "") or not r[0].isdigit() or len(r) < 8:
            continue
        num = lambda v: int(v) if v.isdigit() else 0
        a = agg.setdefault((fil, int(r[0]), r[1].strip()[:90]), [0, 0])
        a[0] += num(r[4])
        a[1] += num(r[7])
    tot = sum(v[0] for v in agg.values()) or 1
    print("total samples", tot, "warp instructions", sum(v[1] for v in agg.values()))
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{v[0]:6d} {100 * v[0] / tot:5.1f}% ins {v[1]:9d} {k[0][:16]}:{k[1]} {k[2]}")


if __name__ == "__main__":
    main()
