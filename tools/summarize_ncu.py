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
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def _csv_rows(text):
    lines = [l for l in text.splitlines() if l.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def launches(path, out, first_epoch=None, last_epoch=None):
    """Per-kernel totals; with first/last epoch (1-based, epochs delimited by
    the trailing Adam launches of each training step) only those epochs count,
    so setup kernels (graph upload, tile build) stay out of the shares."""
    rows = _csv_rows(open(path).read())
    h = rows[0]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    rows = [r for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
    if first_epoch is not None:
        ends, prev_adam = [], False
        for i, r in enumerate(rows):
            is_adam = "adam_kernel" in r[ki]
            if prev_adam and not is_adam:
                ends.append(i)             # first launch after an Adam run = next epoch start
            prev_adam = is_adam
        if prev_adam:
            ends.append(len(rows))
        starts = [0] + ends
        # epoch e (1-based) spans [starts[e-1], ends[e-1]); the first span also holds setup
        rows = rows[starts[int(first_epoch) - 1]:ends[int(last_epoch) - 1]]
    agg = collections.OrderedDict()
    unit = None
    for r in rows:
        unit = r[ui]
        name = re.sub(r"\(.*", "", r[ki])[:90]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    sel = f" epochs {first_epoch}-{last_epoch}" if first_epoch is not None else ""
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised){sel}; unit {unit}",
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
            kk = k if k in idx else next((h for h in idx if h.endswith("." + k)), None)
            if kk is not None:
                e[k] = f"{d[idx[kk]]} {units[idx[kk]]}".strip()
        res.append(e)
    open(out, "w").write(json.dumps(res, indent=1) + "\n")
    for e in res:
        print(e["kernel"], e.get("gpu__time_duration.sum"), "dram", e.get("dram__bytes_read.sum"),
              e.get("dram__bytes_write.sum"), "regs", e.get("launch__registers_per_thread"))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](*sys.argv[2:])
