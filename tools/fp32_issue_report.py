"""Issued vs algorithmic FP32 work per dwell kernel of one ncu --set full report (run here, no
GPU): from the SASS source page, the thread-level (predicated-on) FP32 instructions executed --
FADD/FMUL/FFMA count 1 per lane, the packed FADD2/FFMA2 count 2 (two pixels' operations) --
against the algorithmic work, 6 x the iterations the kernel computes (the
iterations come from the census / stats pass passed in as --iters).

    python tools/fp32_issue_report.py REPORT.ncu-rep --launches 0,3,6,9,12,15,18,21 \\
        --iters 1.62e9,0.61e9,... [--md out.md]
"""
import argparse
import csv
import io
import re
import subprocess

FP1 = re.compile(r"^(@!?U?P\w+\s+)?(FADD|FMUL|FFMA)(\.\S+)?\s")
FP2 = re.compile(r"^(@!?U?P\w+\s+)?(FADD2|FMUL2|FFMA2)(\.\S+)?\s")


def issued(rep, launch):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(launch),
                          "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    name = lines[0].split(",", 1)[1].strip('",')
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ia, isrc = h.index("Address"), h.index("Source")
    ith = h.index("Predicated-On Thread Instructions Executed")
    iex = h.index("Instructions Executed")
    seen, fp, allw = set(), 0, 0
    for r in rows[1:]:
        if len(r) <= ith or r[ia] in seen:
            continue
        try:
            int(r[ia], 16)
        except ValueError:
            continue
        seen.add(r[ia])
        s = r[isrc].strip() + " "
        th = int(float(r[ith] or 0))
        allw += int(float(r[iex] or 0))
        if FP2.match(s):
            fp += 2 * th
        elif FP1.match(s):
            fp += th
    return name, fp, allw


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--launches", required=True)
    ap.add_argument("--iters", required=True)
    ap.add_argument("--labels", default=None)
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    launches = [int(x) for x in a.launches.split(",")]
    iters = [float(x) for x in a.iters.split(",")]
    labels = a.labels.split(",") if a.labels else [str(x) for x in launches]
    out = ["| kernel | iterations | algorithmic FP32 (6/iter) | issued FP32 lane-ops | issued / algorithmic | warp instructions |",
           "|---|---|---|---|---|---|"]
    for lab, l, it in zip(labels, launches, iters):
        name, fp, allw = issued(a.rep, l)
        alg = 6 * it
        out.append(f"| {lab} | {it:.3e} | {alg:.3e} | {fp:.3e} | {fp / alg:.3f} | {allw:.3e} |")
    txt = "\n".join(out)
    print(txt)
    if a.md:
        with open(a.md, "w") as f:
            f.write(f"# Issued vs algorithmic FP32 work per dwell kernel\n\nSource: `{a.rep.split('/')[-1]}` "
                    "(ncu --set full, SASS source page: predicated-on thread instructions; FADD2/FFMA2 "
                    "count 2 per lane). Algorithmic = 6 FP32 instructions x the kernel's iterations "
                    "(`profiles/r02_dwell_census.jsonl`). The excess is chunk overshoot, idle/waiting "
                    "slots, the bisection replay, the escape tests and the pixel-to-c mapping.\n\n" + txt + "\n")


if __name__ == "__main__":
    main()
