"""Summarise an ncu launch list (gpu__time_duration + dram bytes) per kernel class.

    python tools/profile_summary.py gpurun_out/launches.csv profiles/<name>

Writes <name>.md (per-kernel table) and updates profiles/ncu_traffic.json with
the DRAM bytes per launch of each bench.py kernel class (bench.py reads it for
roofline.traffic).
"""
import collections, csv, json, os, sys

CLASS = {"synth_pass": "synth_rowfft", "synth256": "synth_rowfft", "col_pass": "col_residual",
         "col_pass256": "col_residual", "analysis_pass": "rowifft_analysis", "analysis256": "rowifft_analysis",
         "sure_select": "sure_select", "sure_win32": "sure_select", "sure_win_full": "sure_select",
         "sure_select_flagged": "sure_select", "big_keys": "sure_select", "big_range": "sure_select", "row_pass": "finalize"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def main(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.defaultdict(dict)
    name = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        name[r[ii]] = r[ki].split("(")[0].replace("void ", "")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for i, d in per.items():
        n = name[i]
        cnt[n] += 1
        for m, v in d.items():
            agg[n][m] += v
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    lines = ["| kernel | launches | avg us | share | DRAM MB/launch |", "|---|---|---|---|---|"]
    traffic = {}
    cls_bytes = collections.defaultdict(float)
    cls_launch = collections.Counter()
    for n, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        c = cnt[n]
        dram = (a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)) / c
        lines.append(f"| {n} | {c} | {a['gpu__time_duration.sum'] / c * 1e6:.1f} | "
                     f"{a['gpu__time_duration.sum'] / tot:.3f} | {dram / 1e6:.1f} |")
        base = n.split("<")[0]
        cl = CLASS.get(base)
        if cl and "dram__bytes_read.sum" in a:
            cls_bytes[cl] += dram * c
            cls_launch[cl] += c
    for cl in cls_bytes:
        traffic[cl] = cls_bytes[cl] / cls_launch[cl]           # average per launch of the class
    open(out + ".md", "w").write("\n".join(lines) + "\n")
    tpath = os.path.join(os.path.dirname(out), "ncu_traffic.json")
    traffic["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged over all launches "
                        f"of each bench.py kernel class, from {os.path.basename(path)} -> {os.path.basename(out)}.md")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
