"""Per-source-line instruction profile of one kernel launch from an ncu report (run here, no
GPU): ncu's SASS source page (instructions executed per SASS address) joined with the line
table of the library's cubin (nvdisasm -g), aggregated per source line and per opcode class.

    python tools/sass_profile.py REPORT.ncu-rep --launch K [--lib paper_2206_02255_b200/libmandel_b200.so]
           [--top 40] [--json out.json]

Columns: warp-level instructions executed (issue slots), their share, thread-level
predicated-on instructions, FP32-pipe instructions among them.
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess
import tempfile

FP32 = re.compile(r"^(FADD|FMUL|FFMA|FADD2|FMUL2|FFMA2|FMNMX)\b")


def sass_page(rep, launch):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(launch),
                          "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    kname = lines[0].split(",", 1)[1].strip('",')
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ia, isrc, iex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
    ith = h.index("Predicated-On Thread Instructions Executed")
    isamp = h.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in h else None
    stall_cols = [(i, c[len("stall_"):]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    res, seen = [], set()
    for r in rows[1:]:
        if r and r[ia] in seen:  # ncu prints the page once per view: keep the first
            continue
        if r:
            seen.add(r[ia])
        if len(r) <= ith:
            continue
        try:
            st = {c: int(float(r[i] or 0)) for i, c in stall_cols if i < len(r) and r[i] not in ("", "0", "-")}
            samp = int(float(r[isamp] or 0)) if isamp is not None and r[isamp] not in ("", "-") else 0
            res.append((int(r[ia], 16), r[isrc].strip(), int(float(r[iex] or 0)), int(float(r[ith] or 0)), samp, st))
        except ValueError:
            continue
    return kname, res


def line_table(lib, mangled):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    cub = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    start = txt.index(f".text.{mangled}:")
    end = txt.find("//---------------------", start)
    body = txt[start:end if end > 0 else len(txt)]
    table, cur = {}, ("?", 0)
    for ln in body.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            table[int(m.group(1), 16)] = cur
    return table


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--launch", type=int, required=True)
    ap.add_argument("--lib", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "paper_2206_02255_b200", "libmandel_b200.so"))
    ap.add_argument("--mangled", default=None)
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    kname, rows = sass_page(a.rep, a.launch)
    mangled = a.mangled
    if mangled is None:  # demangled "void mandel::k_b200_border_rf<(bool)0>(mandel::LevelArgs)"
        base = re.search(r"mandel::(\w+)<", kname).group(1)
        b = "(bool)1" in kname
        mangled = f"_ZN6mandel{len(base)}{base}ILb{1 if b else 0}EEEvNS_9LevelArgsE"
    table = line_table(a.lib, mangled)
    base_addr = rows[0][0]
    per_line = collections.Counter()
    per_line_fp = collections.Counter()
    per_op = collections.Counter()
    per_line_samp = collections.Counter()
    per_line_stall = collections.defaultdict(collections.Counter)
    stall_tot = collections.Counter()
    tot = fp = samp_tot = 0
    for addr, src, ex, th, samp, st in rows:
        key = table.get(addr - base_addr, ("?", 0))
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        per_line[key] += ex
        per_line_samp[key] += samp
        samp_tot += samp
        for c, v in st.items():
            per_line_stall[key][c] += v
            stall_tot[c] += v
        per_op[op.split(".")[0]] += ex
        tot += ex
        if FP32.match(op):
            per_line_fp[key] += ex
            fp += ex
    print(f"{kname}: {tot:.4e} warp instructions, FP32-pipe {fp / max(tot, 1):.3f}")
    print(f"{'file:line':>24} {'inst':>12} {'share':>7} {'fp32':>7}")
    for key, v in per_line.most_common(a.top):
        print(f"{key[0]:>18}:{key[1]:<5} {v:12.4e} {v / tot:7.3f} {per_line_fp[key] / max(v, 1):7.2f}")
    print("opcodes:", ", ".join(f"{k} {v / tot:.3f}" for k, v in per_op.most_common(25)))
    if samp_tot:
        print(f"stall samples {samp_tot}:", ", ".join(f"{k} {v / samp_tot:.3f}" for k, v in stall_tot.most_common(12)))
        print(f"{'file:line':>24} {'samples':>8} {'share':>7}  top stalls")
        for key, v in per_line_samp.most_common(a.top):
            top = ", ".join(f"{c} {n / max(v, 1):.2f}" for c, n in per_line_stall[key].most_common(4))
            print(f"{key[0]:>18}:{key[1]:<5} {v:8d} {v / samp_tot:7.3f}  {top}")
    if a.json:
        json.dump({"kernel": kname, "total": tot, "fp32": fp,
                   "lines": [[f"{k[0]}:{k[1]}", v, per_line_fp[k]] for k, v in per_line.most_common()],
                   "ops": dict(per_op)}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
