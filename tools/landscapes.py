"""Analytic landscapes of the paper's cost model: the data behind
Fig. "wrf-analytic" (Omega) and Fig. "speedup-analytic" (S_SBR / S_MBR,
P:320-350), whose plotted values are lost in PAPER.md ([FIGURE]), evaluated from
costmodel.py at the paper's GPU (q=128, c=64) and at B200 (q=148 SMs, c=128 FP32
lanes), with the optimal {g, r, B} searched in {2, 4, ..., 1024} as the paper does.
Host only (no GPU).  Also checks the paper's stated readings of those plots against the
model as implemented, and overlays the measured C2 sweeps when given.

    python tools/landscapes.py [--out profiles/r01_landscapes.json] [--md profiles/r01_landscapes.md]
        [--sweep sbr=profiles/r01_sweep_c2_sbr.json ...]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2206_02255_b200 import costmodel as cm  # noqa: E402

NS = [2 ** k for k in range(6, 17)]
BASE = dict(P=0.5, A=512.0, lam=1.0)
GPUS = {"paper_q128_c64": (cm.PAPER_Q, cm.PAPER_C), "b200_q148_c128": (cm.B200_Q, cm.B200_C)}


def best(objective, n, P, A, lam, q, c, **fix):
    sets = {k: ([fix[k]] if k in fix else list(cm.POW2_SPACE)) for k in ("g", "r", "B")}
    (g, r, B), v, _ = cm.grid_search(objective, n, P, A, lam, q, c, sets["g"], sets["r"], sets["B"])
    return (g, r, B), v


def omega_opt(n, P, A, lam, **fix):
    (g, r, B), w = best("work", n, P, A, lam, cm.PAPER_Q, cm.PAPER_C, **fix)
    return {"g": g, "r": r, "B": B, "omega": cm.exhaustive_work(n, A) / w}


def speed_opt(scheme, n, P, A, lam, q, c, **fix):
    (g, r, B), t = best(scheme, n, P, A, lam, q, c, **fix)
    return {"g": g, "r": r, "B": B, "S": cm.exhaustive_time(n, q, c, A) / t}


def e1():
    """Omega rows: Omega(n) varying P, A, lam; optimal g, r, B vs n; Omega(P)
    at four fixed values of g, r and B."""
    out = {"omega_n_vs_P": {}, "omega_n_vs_A": {}, "omega_n_vs_lam": {}, "opt_grb_vs_n": [],
           "omega_P_fixed": {}}
    for P in (0.25, 0.5, 0.75, 0.9):
        out["omega_n_vs_P"][P] = [omega_opt(n, P, BASE["A"], BASE["lam"])["omega"] for n in NS]
    for A in (64.0, 512.0, 4096.0):
        out["omega_n_vs_A"][A] = [omega_opt(n, BASE["P"], A, BASE["lam"])["omega"] for n in NS]
    for lam in (1.0, 100.0, 1e4):
        out["omega_n_vs_lam"][lam] = [omega_opt(n, BASE["P"], BASE["A"], lam)["omega"] for n in NS]
    for n in NS:
        out["opt_grb_vs_n"].append(dict(n=n, **omega_opt(n, **BASE)))
    Ps = [i / 20 for i in range(1, 20)]
    n = 2 ** 14
    for name, vals in (("g", (2, 8, 32, 128)), ("r", (2, 4, 8, 16)), ("B", (2, 8, 32, 128))):
        for v in vals:
            out["omega_P_fixed"][f"{name}={v}"] = [omega_opt(n, P, BASE["A"], BASE["lam"], **{name: v})["omega"]
                                                  for P in Ps]
    out["omega_P_axis"] = Ps
    out["omega_P_n"] = n
    return out


def e2(q, c):
    """Speedup rows at (q, c): S(n) varying lam; S(g), S(r), S(B) at n = 2^15
    (C3's n) with the other two parameters optimal."""
    out = {"S_n_vs_lam": {}, "S_param": {}}
    for lam in (1.0, 100.0, 1e4, 1e6):
        out["S_n_vs_lam"][lam] = {s: [speed_opt(s, n, BASE["P"], BASE["A"], lam, q, c)["S"] for n in NS]
                                  for s in ("sbr", "mbr")}
    n = 2 ** 15
    for name in ("g", "r", "B"):
        vals = [v for v in cm.POW2_SPACE if not (name in ("g", "B") and v > n // 2)]
        out["S_param"][name] = {"axis": vals}
        for lam in (1.0, 1e6):
            for s in ("sbr", "mbr"):
                out["S_param"][name][f"{s},lam={lam:g}"] = [
                    speed_opt(s, n, BASE["P"], BASE["A"], lam, q, c, **{name: v})["S"] for v in vals]
    out["S_param_n"] = n
    return out


def argmax(axis, ys):
    i = max(range(len(ys)), key=lambda k: ys[k])
    return axis[i]


def claims(E1, E2p):
    """The paper's readings of its plots, checked on the model."""
    res = {}
    allw = [w for d in (E1["omega_n_vs_P"], E1["omega_n_vs_A"], E1["omega_n_vs_lam"]) for v in d.values() for w in v]
    res["Omega <= A everywhere (P:244)"] = all(
        w <= A * (1 + 1e-12) for A, ws in E1["omega_n_vs_A"].items() for w in ws) and all(
        w <= BASE["A"] * (1 + 1e-12) for ws in E1["omega_n_vs_P"].values() for w in ws)
    res["Omega: lower P reaches the bound sooner (P:256)"] = all(
        E1["omega_n_vs_P"][0.25][i] >= E1["omega_n_vs_P"][0.9][i] for i in range(len(NS)))
    big = E1["opt_grb_vs_n"][-1]
    res[f"work-optimal r ~ 2 (P:258): r={big['r']} at n=2^16"] = big["r"] == 2
    res[f"work-optimal B ~ 2^3 (P:258): B={big['B']} at n=2^16"] = big["B"] in (4, 8, 16)
    res[f"work-optimal g ~ 2^4 at the largest n (P:258): g={big['g']}"] = big["g"] in (8, 16, 32)
    sp = E2p["S_param"]
    gb_s = argmax(sp["g"]["axis"], sp["g"]["sbr,lam=1"])
    gb_m = argmax(sp["g"]["axis"], sp["g"]["mbr,lam=1"])
    rb_s = argmax(sp["r"]["axis"], sp["r"]["sbr,lam=1"])
    rb_l = argmax(sp["r"]["axis"], sp["r"]["sbr,lam=1e+06"])
    Bb_s = argmax(sp["B"]["axis"], sp["B"]["sbr,lam=1"])
    res[f"S(g): MBR prefers g ~ 2 (P:338): g={gb_m}"] = gb_m <= 4
    res[f"S(g): SBR prefers g ~ 2^5 (P:338): g={gb_s}"] = 16 <= gb_s <= 64
    res[f"S(r): r ~ 2 optimal (P:340): r={rb_s}"] = rb_s == 2
    res[f"S(r): lam=1e6 shifts r right (P:340): r={rb_l}"] = rb_l > rb_s
    res[f"S(B): optimal B ~ 2^5 (P:342): B={Bb_s}"] = 16 <= Bb_s <= 64
    sn = E2p["S_n_vs_lam"][1.0]["sbr"]
    first = next((NS[i] for i in range(len(NS)) if sn[i] > 1.0), None)
    res[f"S(n) > 1 from n >= 2^10 at lam <= 100 (P:336): first n={first}"] = first is not None and first <= 2 ** 10
    return res


def sweep_overlay(paths):
    out = {}
    for spec in paths:
        name, path = spec.split("=", 1)
        rep = json.load(open(path))
        pts = rep["points"]
        meas = {(p["g"], p["r"], p["B"]): p["ms"] for p in pts}
        bm = min(meas, key=meas.get)
        o = {"scheme": rep.get("scheme"), "model_scheme": rep.get("model_scheme"), "t_ex_ms": rep["t_ex_ms"],
             "meas_argmin": list(bm), "meas_min_ms": meas[bm], "meas_speedup_best": rep["t_ex_ms"] / meas[bm],
             "meas_ms_g16r2B32": meas.get((16, 2, 32))}
        for key, m in rep.get("model", {}).items():
            o[key] = {k: m[k] for k in ("pred_argmin", "regret", "spearman", "top5_overlap", "D", "lambda")}
        out[name] = o
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_landscapes.json"))
    ap.add_argument("--md", default=os.path.join(ROOT, "profiles", "r01_landscapes.md"))
    ap.add_argument("--sweep", nargs="*", default=[])
    a = ap.parse_args()
    rep = {"base": BASE, "n_axis": NS, "E1_omega": e1(), "E2_speedup": {}}
    for nm, (q, c) in GPUS.items():
        rep["E2_speedup"][nm] = e2(q, c)
    rep["claims_paper_gpu"] = claims(rep["E1_omega"], rep["E2_speedup"]["paper_q128_c64"])
    rep["claims_b200"] = claims(rep["E1_omega"], rep["E2_speedup"]["b200_q148_c128"])
    rep["measured_c2"] = sweep_overlay(a.sweep)
    with open(a.out, "w") as f:
        json.dump(rep, f, indent=1, default=str)
    write_md(rep, a.md)
    print(open(a.md).read())


def fmt(v):
    return f"{v:.3g}" if isinstance(v, float) else str(v)


def write_md(rep, path):
    L = ["# Cost-model landscapes (NEXT-2): the data of the paper's Omega and speedup figures",
         "",
         "Generated by `tools/landscapes.py` from `paper_2206_02255_b200/costmodel.py` (formulas as printed, "
         "P:112-319; literal tau). Defaults P=0.5, A=512, lambda=1; optimal {g,r,B} searched in {2..1024} "
         "(P:242). Paper GPU q=128, c=64 (P:320); B200 q=148, c=128.", ""]
    E1 = rep["E1_omega"]
    L += ["## Omega(n) with optimal {g,r,B} (Fig. wrf-analytic, row 1)", "",
          "| n | " + " | ".join(f"P={p}" for p in E1["omega_n_vs_P"]) + " | "
          + " | ".join(f"A={int(float(x))}" for x in E1["omega_n_vs_A"]) + " | "
          + " | ".join(f"lam={float(x):g}" for x in E1["omega_n_vs_lam"]) + " |",
          "|---" * (1 + len(E1["omega_n_vs_P"]) + len(E1["omega_n_vs_A"]) + len(E1["omega_n_vs_lam"])) + "|"]
    for i, n in enumerate(rep["n_axis"]):
        cells = [fmt(v[i]) for v in E1["omega_n_vs_P"].values()] + [fmt(v[i]) for v in E1["omega_n_vs_A"].values()] \
            + [fmt(v[i]) for v in E1["omega_n_vs_lam"].values()]
        L.append(f"| 2^{int(math.log2(n))} | " + " | ".join(cells) + " |")
    L += ["", "## Work-optimal {g, r, B} vs n (row 2)", "", "| n | g | r | B | Omega |", "|---|---|---|---|---|"]
    for o in E1["opt_grb_vs_n"]:
        L.append(f"| 2^{int(math.log2(o['n']))} | {o['g']} | {o['r']} | {o['B']} | {fmt(o['omega'])} |")
    for nm, E2 in rep["E2_speedup"].items():
        L += ["", f"## Speedup S(n), optimal {{g,r,B}}, {nm} (Fig. speedup-analytic, row 1)", "",
              "| n | " + " | ".join(f"{s} lam={float(l):g}" for l in E2["S_n_vs_lam"] for s in ("sbr", "mbr")) + " |",
              "|---" * (1 + 2 * len(E2["S_n_vs_lam"])) + "|"]
        for i, n in enumerate(rep["n_axis"]):
            L.append(f"| 2^{int(math.log2(n))} | " + " | ".join(
                fmt(E2["S_n_vs_lam"][l][s][i]) for l in E2["S_n_vs_lam"] for s in ("sbr", "mbr")) + " |")
        L += ["", f"S(g), S(r), S(B) at n=2^15 (rows 2-4), {nm}: the argmax per curve", "",
              "| param | sbr lam=1 | mbr lam=1 | sbr lam=1e6 | mbr lam=1e6 |", "|---|---|---|---|---|"]
        for p, d in E2["S_param"].items():
            L.append(f"| {p} | " + " | ".join(
                f"{argmax(d['axis'], d[k])} (S={fmt(max(d[k]))})" for k in
                ("sbr,lam=1", "mbr,lam=1", "sbr,lam=1e+06", "mbr,lam=1e+06")) + " |")
    for which in ("claims_paper_gpu", "claims_b200"):
        L += ["", f"## The paper's readings of its plots, checked on the model ({which[7:]})", ""]
        for k, v in rep[which].items():
            L.append(f"- {'holds' if v else 'does NOT hold'}: {k}")
    if rep["measured_c2"]:
        L += ["", "## Measured C2 sweeps on one B200 (n=8192, maxdwell 2048) vs the calibrated model", "",
              "| run | measured argmin | min ms | best speedup vs Ex | model (A, tau) | predicted argmin | regret | Spearman | top-5 overlap |",
              "|---|---|---|---|---|---|---|---|---|"]
        for nm, o in rep["measured_c2"].items():
            for key, m in o.items():
                if isinstance(m, dict):
                    L.append(f"| {nm} | {o['meas_argmin']} | {fmt(o['meas_min_ms'])} | {fmt(o['meas_speedup_best'])} | "
                             f"{key} | {m['pred_argmin']} | {fmt(m['regret'])} | {fmt(m['spearman'])} | {m['top5_overlap']} |")
    with open(path, "w") as f:
        f.write("\n".join(L) + "\n")


if __name__ == "__main__":
    main()
