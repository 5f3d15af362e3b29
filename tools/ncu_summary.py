"""Summarise an ncu --set full report into the evidence north_star asks for (run here, no GPU):

  * FP32-pipe utilisation    sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active
                             (+ sm__pipe_fma_cycles_active) on the dwell kernels;
  * HBM traffic and GB/s     dram__bytes_read.sum + dram__bytes_write.sum per launch, / duration,
                             on fill and classification (list compaction) kernels;
  * warp execution efficiency smsp__thread_inst_executed_per_inst_executed.ratio / 32;
  * issue-slot use            smsp__issue_active.avg.pct_of_peak_sustained_active.

    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep --title "..." --md profiles/x.md \
        [--traffic-key C3:b200 --traffic-json profiles/ncu_traffic.json]

--traffic-json merges {"<key>:<kernel kind>": bytes per launch} for bench.py's roofline.traffic.
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess

M = {
    "time_ms": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "fma_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "fma_cyc_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "thr_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "inst": "smsp__inst_executed.sum",
}
SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def kind_of(name: str) -> str:
    m = re.search(r"k3?_(b200_border_rf|b200_border|b200_classify|b200_leaf_rf|b200_leaf|fill|sbr_level|sbr_leaf|"
                  r"exhaustive\w*|init|surface_rf|surface|classify|leaf_rf|leaf)", name)
    if not m:
        return name[:40]
    return m.group(1)[:-3] if m.group(1).endswith("_rf") else m.group(1)  # bench.py kind names


def load(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {"name": r[hdr.index("Kernel Name")]}
        for k, col in M.items():
            if col not in hdr:
                d[k] = None
                continue
            i = hdr.index(col)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                d[k] = None
                continue
            d[k] = v * SCALE.get(units[i], 1.0) if k in ("time_ms", "dram_rd", "dram_wr") else v
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--title", default="")
    ap.add_argument("--md", required=True)
    ap.add_argument("--traffic-key")
    ap.add_argument("--traffic-json")
    a = ap.parse_args()
    ks = load(a.rep)
    lines = [f"# ncu summary: {a.title}", "", f"Source: `{os.path.basename(a.rep)}` (`ncu --set full "
             "--clock-control none`; per-launch, cold-cache, serialised replays).", "",
             "| # | kernel | ms | DRAM rd+wr MB | DRAM GB/s | FP32 pipe % (inst) | warp exec eff | issue active % "
             "| warps active % | regs | grid |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for i, k in enumerate(ks):
        by = (k["dram_rd"] or 0) + (k["dram_wr"] or 0)
        gbs = by / (k["time_ms"] * 1e-3) / 1e9 if k["time_ms"] else 0.0
        eff = (k["thr_per_inst"] or 0) / 32.0
        lines.append(f"| {i} | {kind_of(k['name'])} | {k['time_ms']:.3f} | {by / 1e6:.1f} | {gbs:.0f} | "
                     f"{(k['fma_pct'] or 0):.1f} | {eff:.3f} | {(k['issue_pct'] or 0):.1f} | "
                     f"{(k['warps_pct'] or 0):.1f} | {int(k['regs'] or 0)} | {int(k['grid'] or 0)} |")
        traffic.setdefault(kind_of(k["name"]), []).append(by)
    lines.append("")
    lines.append("FP32 pipe % = sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active; warp exec eff = "
                 "smsp__thread_inst_executed_per_inst_executed.ratio / 32.")
    with open(a.md, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if a.traffic_json and a.traffic_key:
        cur = {}
        if os.path.exists(a.traffic_json):
            cur = json.load(open(a.traffic_json))
        for kind, v in traffic.items():
            cur[f"{a.traffic_key}:{kind}"] = sum(v) / len(v)
        with open(a.traffic_json, "w") as f:
            json.dump(cur, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
