"""Summarise ncu outputs for profiles/.

  python tools/ncu_summary.py rep <file.ncu-rep> [--json out.json]   # --set full capture
  python tools/ncu_summary.py launches <launches.csv>                 # gpu__time_duration launch list
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]


def short(name):
    return name.split("(")[0].replace("void ", "").replace("exmy::", "")


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k in KEYS:
            if k in hdr:
                v = r[hdr.index(k)].replace(",", "")
                try:
                    d[k] = float(v)
                except ValueError:
                    d[k] = v
                d[k + ".unit"] = units[hdr.index(k)]
        stalls = []
        for i, h in enumerate(hdr):
            if "smsp__average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio") and "not_issued" not in h:
                try:
                    stalls.append((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                                   float(r[i])))
                except ValueError:
                    pass
        stalls.sort(key=lambda t: -t[1])
        d["top_stalls_per_issue"] = stalls[:5]
        rb = d.get("dram__bytes_read.sum", 0.0)
        wb = d.get("dram__bytes_write.sum", 0.0)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rb *= scale.get(d.get("dram__bytes_read.sum.unit", "byte"), 1)
        wb *= scale.get(d.get("dram__bytes_write.sum.unit", "byte"), 1)
        d["dram_bytes_total"] = rb + wb
        res.append(d)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            agg[short(r[ki])[:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = []
    for k, v in sorted(agg.items(), key=lambda t: -sum(t[1])):
        lines.append({"kernel": k, "launches": len(v), "avg_ns": sum(v) / len(v), "share": sum(v) / tot})
    return lines


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    data = rep(path) if mode == "rep" else launches(path)
    if "--json" in sys.argv:
        json.dump(data, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    if mode == "rep":
        for d in data:
            print(f"{d['kernel']:40s} {d['gpu__time_duration.sum']:9.1f}{d['gpu__time_duration.sum.unit']} "
                  f"dram={d['dram_bytes_total'] / 1e6:8.1f} MB issue={d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):5.1f}% "
                  f"warps={d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):5.1f}% "
                  f"regs={d.get('launch__registers_per_thread', 0):.0f} stalls={d['top_stalls_per_issue'][:3]}")
    else:
        for d in data:
            print(f"{d['kernel']:70s} n={d['launches']:4d} avg={d['avg_ns'] / 1e3:9.1f} us share={100 * d['share']:5.1f}%")
