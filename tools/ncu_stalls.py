"""Print key metrics + warp stall breakdown per kernel of an ncu report."""
import csv
import io
import subprocess
import sys


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
    for r in rows[2:]:
        print("==", r[hdr.index("Kernel Name")][:90])
        for k in keys:
            if k in hdr:
                print(f"   {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
        st = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled_")
              or (h.startswith("smsp__warp_issue_stalled_") and h.endswith("_per_warp_active.pct"))]
        vals = []
        for h, v in st:
            try:
                vals.append((float(v), h))
            except ValueError:
                pass
        for v, h in sorted(vals, reverse=True)[:8]:
            print(f"   stall {h} = {v}")


if __name__ == "__main__":
    main(sys.argv[1])
