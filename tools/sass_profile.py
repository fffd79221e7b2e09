"""Per-instruction SASS execution profile of one kernel from an ncu report
(source page, SASS view), grouped by opcode and by code region.

  python tools/sass_profile.py <report.ncu-rep> <kernel regex> [elements]

Regions are contiguous address ranges split at the kernel's hottest basic
blocks; `elements` (optional) divides thread-instruction counts into
per-element figures (e.g. the quantized elements of a K1 launch)."""
import collections
import csv
import io
import re
import subprocess
import sys


def load(rep, kregex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kregex}"], capture_output=True, text=True).stdout
    kernels, cur = [], None
    for line in out.splitlines():
        if line.startswith('"Kernel Name"'):
            cur = {"name": next(csv.reader(io.StringIO(line)))[1], "rows": []}
            kernels.append(cur)
        elif cur is not None and line.startswith('"0x'):
            cur["rows"].append(next(csv.reader(io.StringIO(line))))
    return kernels


def main(rep, kregex, elements=None):
    for k in load(rep, kregex):
        ops = collections.Counter()
        total_thr = 0
        for r in k["rows"]:
            src = r[1].strip()
            m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src)
            op = m.group(2) if m else "?"
            thr = int(r[6] or 0)          # thread instructions executed
            ops[op] += thr
            total_thr += thr
        print(f"== {k['name']}")
        print(f"thread instructions: {total_thr:.4g}" +
              (f"  per element: {total_thr / float(elements):.1f}" if elements else ""))
        for op, n in ops.most_common(25):
            print(f"  {op:12s} {n / total_thr * 100:5.1f}%" + (f"  {n / float(elements):6.2f}/elem" if elements else ""))


if __name__ == "__main__":
    main(*sys.argv[1:])
