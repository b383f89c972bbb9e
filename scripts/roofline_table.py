"""Hierarchical roofline table (HBM / L2 / L1 traffic of
every kernel) from an ncu metrics capture of one solve.

Capture (GPU box, one solve without the graph so ncu sees every kernel):
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,\
l1tex__t_bytes.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,\
sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
      --clock-control none --csv --log-file <csv> python bench.py --steps 1 --warmup 0 --no-cpu --no-fp64 \
      --no-kernels --no-graph --no-extra [--variant d_mg | --dim 2 --nodes 8193]

Summarise:  python scripts/roofline_table.py <csv> <peaks.txt> [title] > table.md
The per-launch times are serialised and cold-cache (ncu), so they explain
shares and bandwidths per level, not the graph-launched solve time.
"""
import csv
import io
import json
import os
import re
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_peaks(path):
    p = {}
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        p["hbm"] = float(json.load(f)["hbm_gbs"])
    if path and os.path.exists(path):
        for line in open(path):
            t = line.split()
            if len(t) >= 2 and t[0].endswith(("_gbs", "_tflops", "_nontensor")):
                try:
                    p[t[0]] = float(t[1])
                except ValueError:
                    pass
    return p


def short(name):
    name = re.sub(r"\(.*\)$", "", name)
    name = name.replace("mpmg_impl::<unnamed>::", "").replace("mpmg_dev::", "").replace("coarse_detail::", "")
    return name


def main():
    path = sys.argv[1]
    peaks = load_peaks(sys.argv[2] if len(sys.argv) > 2 else None)
    title = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(path)
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    per = OrderedDict()  # launch id -> dict(name, grid, metrics)
    for r in rows:
        key = r["ID"]
        d = per.setdefault(key, {"name": r["Kernel Name"], "grid": r.get("Grid Size", ""), "m": {}})
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
                 "msecond": 1e-3, "second": 1.0, "%": 1.0}.get(unit, 1.0)
        d["m"][r["Metric Name"]] = v * scale
    groups = OrderedDict()
    for d in per.values():
        k = (short(d["name"]), d["grid"])
        g = groups.setdefault(k, {"n": 0, "t": 0.0, "dram": 0.0, "l2": 0.0, "l1": 0.0, "fma": 0.0, "fp64": 0.0})
        m = d["m"]
        g["n"] += 1
        g["t"] += m.get("gpu__time_duration.sum", 0.0)
        g["dram"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        g["l2"] += m.get("lts__t_bytes.sum", 0.0)
        g["l1"] += m.get("l1tex__t_bytes.sum", 0.0)
        g["fma"] += m.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
        g["fp64"] += m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
    total = sum(g["t"] for g in groups.values()) or 1.0
    l2p, l1p = peaks.get("l2_read_gbs"), peaks.get("smem_read_gbs")
    print(f"## {title}\n")
    print(f"Peaks (measured on this B200): HBM {peaks['hbm']:.0f} GB/s (MEASURED_PEAKS.json), "
          f"L2 {l2p or float('nan'):.0f} GB/s, L1/shared {l1p or float('nan'):.0f} GB/s "
          f"(scripts/probe_peaks.cu).\n")
    print("| kernel | grid | launches | share | us/launch | HBM MB | HBM GB/s (% peak) | L2 MB | L2 GB/s (% peak) "
          "| L1 MB | L1 GB/s (% peak) | FMA pipe % | FP64 pipe % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    out = []
    for (name, grid), g in sorted(groups.items(), key=lambda kv: -kv[1]["t"]):
        n, t = g["n"], g["t"] / g["n"]
        if g["t"] / total < 0.003:
            continue
        dram, l2, l1 = g["dram"] / n, g["l2"] / n, g["l1"] / n
        bw = lambda b: b / t / 1e9 if t > 0 else 0.0
        pc = lambda x, p: f"{x:.0f} ({100 * x / p:.0f}%)" if p else f"{x:.0f}"
        print(f"| `{name[:70]}` | {grid} | {n} | {100 * g['t'] / total:.1f}% | {t * 1e6:.2f} | {dram / 1e6:.1f} | "
              f"{pc(bw(dram), peaks['hbm'])} | {l2 / 1e6:.1f} | {pc(bw(l2), l2p)} | {l1 / 1e6:.1f} | {pc(bw(l1), l1p)} | "
              f"{g['fma'] / n:.0f} | {g['fp64'] / n:.0f} |")
        out.append(dict(kernel=name, grid=grid, launches=n, us=t * 1e6, dram_bytes=dram, l2_bytes=l2, l1_bytes=l1,
                        fma_pipe_pct=g["fma"] / n, fp64_pipe_pct=g["fp64"] / n, share=g["t"] / total))
    if len(sys.argv) > 4:
        with open(sys.argv[4], "w") as f:
            json.dump({"title": title, "peaks": peaks, "kernels": out}, f, indent=1)


if __name__ == "__main__":
    main()
