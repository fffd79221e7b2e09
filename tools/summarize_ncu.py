"""Summarise ncu outputs into profiles/ (run in the build container).

  python tools/summarize_ncu.py launches <launches.csv> <out.txt> [--last-epochs N --epoch-marker REGEX]
  python tools/summarize_ncu.py full <report.ncu-rep> <out.json>
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

FULL_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def _csv_rows(text):
    lines = [l for l in text.splitlines() if l.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def launches(path, out):
    rows = _csv_rows(open(path).read())
    h = rows[0]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.OrderedDict()
    unit = None
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        unit = r[ui]
        name = re.sub(r"\(.*", "", r[ki])[:90]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised); unit {unit}",
             "kernel | launches | total | share"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k} | {v[0]} | {v[1]:.0f} | {v[1] / tot:.3f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:20]))


def full(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = _csv_rows(txt)
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {x: i for i, x in enumerate(hdr)}
    res = []
    for d in data:
        e = {"kernel": re.sub(r"\(.*", "", d[idx["Kernel Name"]])}
        for k in FULL_KEYS:
            if k in idx:
                e[k] = f"{d[idx[k]]} {units[idx[k]]}".strip()
        res.append(e)
    open(out, "w").write(json.dumps(res, indent=1) + "\n")
    for e in res:
        print(e["kernel"], e.get("gpu__time_duration.sum"), "dram", e.get("dram__bytes_read.sum"),
              e.get("dram__bytes_write.sum"), "regs", e.get("launch__registers_per_thread"))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
