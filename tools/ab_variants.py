"""A/B of compile-time variants of libmandel_b200.so (dev tool).

Build here (CPU, nvcc cross-compiles; the .so files travel to the GPU box in build/variants/):
    python tools/ab_variants.py build  NAME=DEF1,DEF2 NAME2=DEF3 ...      (DEF: MANDEL_ knob w/o prefix)
Run on the GPU box:
    python tools/ab_variants.py run [--workloads C3,C5,C3r8] [--rounds 3] [--reps 5] [--check] NAME ...

Each (round, variant) runs in its own process (the library is loaded once per process through
MANDEL_B200_LIB): device time per ASK step (CUDA events, L2 flushed between reps) for each
workload -- C3r8 = the heaviest rank's tiles of an 8-way LPT deal on exact tile costs -- and,
with --check, the full image's tile digests against the oracle golden files (bit-exactness).
Prints one JSON line per (round, variant, workload) and a summary (median over rounds).
"""
import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "build", "variants")


def so_path(name):
    return os.path.join(VDIR, f"libmandel_{name}.so")


def cmd_build(specs):
    from paper_2206_02255_b200 import build
    os.makedirs(VDIR, exist_ok=True)
    import concurrent.futures as cf
    jobs = {}
    with cf.ThreadPoolExecutor(4) as ex:
        for s in specs:
            name, _, defs = s.partition("=")
            dl = ["MANDEL_" + d for d in defs.split(",") if d]
            jobs[name] = ex.submit(build.build, out=so_path(name), defines=dl)
        for name, f in jobs.items():
            print(name, f.result())


def worker(name, workloads, reps, check):
    os.environ["MANDEL_B200_LIB"] = so_path(name) if name != "base" else ""
    import torch
    import paper_2206_02255_b200 as mb
    from paper_2206_02255_b200 import deal
    import workloads as W
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for wl in workloads:
        wname, _, share = wl.partition("r")
        w = W.CONFIGS[wname]
        out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
        ws = mb.workspace(w.n, w.g, w.r, w.B)
        tiles = None
        dev = share.endswith("d") or share.endswith("n")  # C3r8d: the same rank through mandel_ask_dtiles
        tcm = "sampled" if share.endswith("d") else False  # + sampled costs; C3r8n: without counters
        share = share.rstrip("dn")
        if share:
            mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tile_cost=True)
            exact = mb.tile_costs(ws, w.g)
            parts = deal.deal("lpt", w.g, int(share), exact)
            tiles = max(parts, key=lambda p: sum(exact[k] for k in p))
        if dev:
            dt = torch.tensor(tiles, dtype=torch.int32, device="cuda")
            dn = torch.tensor([len(tiles)], dtype=torch.int32, device="cuda")
            f = lambda: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws,  # noqa: E731
                               dtiles=(dt, dn), tile_cost=tcm)
        else:
            f = lambda: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=tiles)  # noqa: E731
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            f()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        res = {"variant": name, "w": wl, "ms": statistics.median(ts), "ms_min": min(ts)}
        if dev:
            mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, dtiles=(dt, dn), tile_cost=tcm,
                   timing=True)
        else:
            mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=tiles, timing=True)
        torch.cuda.synchronize()
        kt, lv = {}, {}
        for k in mb.kernel_times():
            kt[k["kind"]] = kt.get(k["kind"], 0.0) + k["ms"]
            if k["kind"] in ("b200_border", "b200_classify", "b200_leaf"):
                lv[f"{k['kind'][5:]}{k['level']}"] = round(k["ms"], 4)
        res["kernels"] = {k: round(v, 4) for k, v in kt.items()}
        res["levels"] = lv
        if check and not share:
            from oracle import cache
            rec = cache.tile_records(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
            f()
            torch.cuda.synchronize()
            d0 = w.n // w.g
            bad = 0
            for gy in range(w.g):
                band = out[gy * d0:(gy + 1) * d0].cpu().numpy()
                for gx in range(w.g):
                    t = band[:, gx * d0:(gx + 1) * d0].copy()
                    bad += hashlib.sha256(t.astype("<i4").tobytes()).hexdigest() != rec["tiles"][gy * w.g + gx]["sha256"]
            res["tiles_differing_from_oracle"] = bad
        print(json.dumps(res), flush=True)


def cmd_run(a):
    rows = []
    for rnd in range(a.rounds):
        for name in a.names:
            p = subprocess.run([sys.executable, __file__, "_worker", name, a.workloads, str(a.reps),
                                "1" if (a.check and rnd == 0) else "0"], capture_output=True, text=True)
            for ln in p.stdout.splitlines():
                if ln.startswith("{"):
                    d = json.loads(ln)
                    d["round"] = rnd
                    rows.append(d)
                    print(json.dumps(d), flush=True)
            if p.returncode:
                print(f"[{name}] rc={p.returncode}: {p.stderr[-2000:]}", flush=True)
    print("summary (median over rounds, ms):")
    for wl in a.workloads.split(","):
        line = []
        for name in a.names:
            v = [r["ms"] for r in rows if r["variant"] == name and r["w"] == wl]
            if v:
                line.append(f"{name} {statistics.median(v):.3f}")
        print(f"  {wl}: " + " | ".join(line), flush=True)


def main():
    if sys.argv[1] == "_worker":
        worker(sys.argv[2], sys.argv[3].split(","), int(sys.argv[4]), sys.argv[5] == "1")
        return
    if sys.argv[1] == "build":
        cmd_build(sys.argv[2:])
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd")
    ap.add_argument("names", nargs="+")
    ap.add_argument("--workloads", default="C3,C5,C3r8")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check", action="store_true")
    cmd_run(ap.parse_args())


if __name__ == "__main__":
    main()
