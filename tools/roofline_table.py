"""Per-kernel roofline table (markdown) from a bench JSON line.
  python tools/roofline_table.py profiles/r1_bench_v10_reddit.json [...]"""
import json
import sys


def table(path):
    b = json.loads(open(path).read().strip().splitlines()[-1])
    ms = b["ms_per_step"]
    steps = b["steps"]
    kr = b.get("kernel_rooflines", {})
    out = [f"### {b['config']['workload']}",
           f"epoch {ms:.2f} ms (device, CUDA events), e2e {b['e2e']['value'] * 1e3:.1f} ms, "
           f"clocks {b['clocks'].get('sm_mhz')} MHz {b['clocks'].get('reasons')}", "",
           "| kernel class | ms / epoch | share | achieved | bound | fraction |", "|---|---|---|---|---|---|"]
    roof = b.get("roofline") or {}
    for k, v in sorted(b["kernels"].items(), key=lambda kv: -kv[1]["ms"]):
        per = v["ms"] / steps
        r = roof if (roof and roof.get("l1_datapath") is not None and k.startswith("spmm") and k not in kr) else kr.get(k)
        if r is not None and r.get("l1_datapath") is not None:
            dp = r["l1_datapath"]
            tiled = k == "spmm_tiled"
            ach = (f"{r['achieved']:.0f} GB/s compulsory; {dp.get('gathered_gbps', 0):.0f} GB/s gathered"
                   + (f" (ncu l1tex {dp.get('ncu_l1tex_pct_elapsed')} % of peak)" if tiled else ""))
            bound = "smem datapath" if tiled else "L2 gather"
            frac = f"{r['frac']:.3f} of HBM; {dp.get('frac', 0):.2f} of the smem-datapath model"
        elif r is None and k == "gemm" and roof and roof.get("unit") == "TFLOP/s":
            r = roof
        if r is not None and r.get("l1_datapath") is not None:
            pass
        elif r is not None:
            if r.get("unit") == "TFLOP/s":
                ach = f"{r['achieved']:.0f} TF/s fp32-equiv ({r.get('tf32_mma_tflops', 0):.0f} TF/s TF32 MMA)"
                bound, frac = "tensor (3xTF32)", f"{r['frac']:.2f}"
                if r.get("hbm_frac") is not None:
                    ach += f"; {r['hbm_gbps']:.0f} GB/s compulsory"
                    frac += f" of tensor; {r['hbm_frac']:.2f} of HBM"
                    if r["hbm_frac"] > r["frac"]:
                        bound = "HBM (narrow K) / tensor"
            elif "philox_frac" in r:
                ach = f"{r['achieved']:.0f} GB/s, {r['philox_gelem_s']:.0f} G elem/s"
                bound, frac = "Philox issue rate", f"{r['philox_frac']:.2f} of 414 G/s"
            elif "gathered_gbps" in r:
                ach = f"{r['gathered_gbps']:.0f} GB/s gathered"
                bound, frac = "L2 / smem gather", f"{r['frac']:.3f} HBM"
            else:
                ach = f"{r['achieved']:.0f} GB/s"
                bound, frac = "HBM", f"{r['frac']:.2f}"
        else:
            ach, bound, frac = f"{v.get('gbps', 0):.0f} GB/s", "", ""
        out.append(f"| {k} | {per:.2f} | {per / ms:.2f} | {ach} | {bound} | {frac} |")
    return "\n".join(out)


if __name__ == "__main__":
    print("\n\n".join(table(p) for p in sys.argv[1:]))
