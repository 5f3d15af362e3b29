"""bench.py -- ASK Mandelbrot throughput on B200 (BASELINE.json metric, config 3 by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3] [--scheme b200]
                    [--deal costrank] [--impl ours|reference]

One step = one pass of the whole hot path over the workload: mandel_ask over this rank's
level-0 tiles (init, every level's border + classify + fill, leaves), i.e. the full n x n
dwell image when N = 1.  Inputs (region, n, maxdwell, g, r, B, tile list) are scalars; the
output image (4 GiB at n = 32768) is far larger than L2 and every step rewrites all of
it; an explicit 256 MiB L2 flush also runs between timed steps, outside the per-step events.

N > 1: one process per GPU (torchrun), NCCL process group; level-0 tiles are dealt
longest-first (LPT) on the device: every timed step renders the rank's tiles with per-tile cost
counters, all-reduces the g*g counters and computes the next step's deal (mandel_deal_lpt), so
the plan is charged to every step; the first, untimed step is dealt on an n/32, maxdwell/8
preview.  No collective touches the image on the data path; the time is the max over ranks of
the device time.
MANDEL_DIST_BACKEND=gloo (test only): gloo process group with CPU-side collectives and every
rank on cuda:(LOCAL_RANK mod device count), so the N > 1 control flow can be exercised on a
one-GPU box (ranks then share the GPU: the times are not scaling numbers).

--impl reference: the CPU oracle (oracle/) on the box's host cores on a bounded sample of
the same workload (the reference arm of this tier), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "Mpixel/s & Giter/s, n=32768 ASK, 1/2/4/8 B200; speedup vs exhaustive; % FP32 peak"
FLOPS_PER_ITER = 6          # FP32 instructions per dwell iteration: 3 FMUL + 2 FADD + 1 FFMA(xy, 2, ci)
PAPER_OPS_PER_ITER = 7      # the literal step's 3 FMUL + 4 FADD (R4; R4' fuses (xy+xy)+ci exactly)
N_SM, LANES = 148, 128      # B200: FP32 lanes per SM (one FADD/FMUL per lane per clock)
L2_FLUSH_BYTES = 256 << 20


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------ CPU oracle
def _oracle_tile(args):
    import oracle
    region, n, md, g, r, B, t = args
    t0 = time.perf_counter()
    img, st = oracle.ask_tile(region, n, md, g, r, B, t)
    return t, time.perf_counter() - t0, sum(s["border_iters"] + s["leaf_iters"] for s in st)


def cpu_oracle_sample(w: W.Workload, budget_s: float = 15.0, seed: int = W.SEED):
    """The oracle as it stands (single-threaded C recursion per level-0 tile), one process
    per host core over a seeded random sample of the workload's tiles."""
    import multiprocessing as mp
    import random
    import oracle
    oracle.build()
    cores = len(os.sched_getaffinity(0))
    order = list(range(w.g * w.g))
    random.Random(seed).shuffle(order)
    # bounded sample: ~budget_s of CPU work per core at ~0.5 s per tile on average
    k = min(len(order), max(4, int(cores * budget_s / 2.0)))
    sample = order[:k]
    t0 = time.perf_counter()
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        res = pool.map(_oracle_tile, [(w.region, w.n, w.maxdwell, w.g, w.r, w.B, t) for t in sample],
                       chunksize=1)
    wall = time.perf_counter() - t0
    px = k * (w.n // w.g) ** 2
    iters = sum(x[2] for x in res)
    return {"value": px / wall / 1e6, "unit": "Mpixel/s", "cores": cores, "kind": "oracle",
            "sample": f"{k} of {w.g * w.g} level-0 tiles of {w.name} (seeded random), one oracle "
                      f"process per core, wall {wall:.2f}s, {iters:.3e} executed iterations",
            "wall_s": wall, "giter_s": iters / wall / 1e9}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    w = W.CONFIGS[args.workload]
    vals = []
    last = None
    for i in range(args.warmup + args.steps):
        last = cpu_oracle_sample(w, budget_s=args.ref_budget, seed=W.SEED + i)
        if i >= args.warmup:
            vals.append(last["wall_s"])
    px = float(last["value"]) * last["wall_s"]  # Mpixel per step sample
    ms = 1e3 * sum(vals) / len(vals)
    value = px / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config(w, args, world),
            "cpu_baseline": {k: last[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": value, "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    line["cpu_baseline"]["value"] = value
    print(json.dumps(line), flush=True)


def _config(w: W.Workload, args, world: int):
    return {"workload": f"{w.name}: Mandelbrot n={w.n} maxdwell={w.maxdwell} region={list(w.region)} "
                        f"ASK g={w.g} r={w.r} B={w.B}",
            "n": w.n, "maxdwell": w.maxdwell, "g": w.g, "r": w.r, "B": w.B, "region": list(w.region),
            "scheme": args.scheme, "deal": "lpt (device)" if world > 1 else "all tiles",
            "deal_plan": ("inside the timed steps, every 3rd step (multigpu.SAMPLE_EVERY): sampled per-tile "
                          "cost counters of that step's render (1/64 pixel lattice, dwell + 64 per pixel), then "
                          "on a side stream overlapping the next step's render: NCCL all-reduce of the g*g "
                          "counters and the device LPT deal (mandel_deal_lpt) of the step after next, which waits "
                          "for it on the main stream; the other steps render without counters; the first steps "
                          "are dealt on an n/32, maxdwell/8 preview")
            if world > 1 else None,
            "parallelism": f"tiles{world}",
            "l2": "output image 4*n^2 B >> 126 MB L2, rewritten every step; plus a 256 MiB L2 flush "
                  "between timed steps outside the per-step events"}


# ------------------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C3", choices=sorted(W.CONFIGS))
    ap.add_argument("--scheme", default="b200", choices=["b200", "sbr", "mbr"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the N>1 verification gather")
    ap.add_argument("--ref-budget", type=float, default=12.0)
    args = ap.parse_args()

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2206_02255_b200 as mb
    from paper_2206_02255_b200 import multigpu

    backend = os.environ.get("MANDEL_DIST_BACKEND", "nccl")
    if backend not in ("nccl", "gloo"):
        raise SystemExit(f"MANDEL_DIST_BACKEND={backend}: expected nccl or gloo")
    if backend == "gloo":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # device of collective tensors
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    w = W.CONFIGS[args.workload]
    n = w.n

    # ---- partition.  N > 1: a device-resident LPT deal of the level-0 tiles
    # (multigpu.DevicePlan).  Every SAMPLE_EVERY-th timed step (3) renders this rank's tiles
    # with sampled per-tile cost counters (MANDEL_FLAG_TILE_COST_SAMPLED) and hands them to a
    # side stream, which all-reduces them across ranks and re-deals on the device
    # (mandel_deal_lpt) for the step after next while the next step renders; the other steps
    # render without counters.  The plan is inside the timed region's wall time (its events
    # sit on the main stream, which waits for the plan a step uses), off the critical path.
    # The first steps are dealt on an n/32, maxdwell/8 preview.
    out = torch.empty((n, n), dtype=torch.int32, device=dev)
    ws = mb.workspace(n, w.g, w.r, w.B, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    plan = None
    if world > 1:
        plan = multigpu.DevicePlan(w, world, rank, dev)
        costs0 = torch.zeros(w.g * w.g, dtype=torch.int64, device=dev)
        plan.preview_costs(costs0)
        plan.deal(costs0, both=True)

    def allreduce_costs(t):
        if backend == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        else:  # gloo test mode: host-side collective
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM)
            t.copy_(h)

    # ---- per-kernel algorithmic work from one untimed counter pass (deterministic)
    if plan is None:
        mb.ask(w.region, n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, scheme=args.scheme, stats=True)
    else:  # converge the deal first (the timed steps run the steady state), then count
        for _ in range(4):
            plan.step(out, ws, allreduce_costs)
        torch.cuda.synchronize()
        mb.ask(w.region, n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, dtiles=(plan.tiles, plan.count),
               scheme=args.scheme, stats=True)
    lstats = mb.ask_stats(ws)
    border_iters = sum(s["border_iters"] for s in lstats)
    leaf_iters = sum(s["leaf_iters"] for s in lstats)
    exec_iters = border_iters + leaf_iters

    # timed steps: events around the leaf kernel only (the roofline's dominant kernel, timed
    # live in the timed region); event nodes between every pair of kernels would cut the level
    # chain's programmatic-dependent-launch edges.  The full per-kernel breakdown comes from
    # separate calls after the timed region.
    def step(timing="leaf"):
        if plan is None:
            mb.ask(w.region, n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, scheme=args.scheme, timing=timing)
        else:
            plan.step(out, ws, allreduce_costs, timing=timing)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    kernels_per_step = mb.kernel_count(n, w.g, w.r, w.B, args.scheme)
    plan_steps0 = plan.n_steps if plan is not None else 0

    stream = torch.cuda.current_stream()
    step_ms, ktime = [], {}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush, outside the events
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            for kt in mb.kernel_times():
                ktime.setdefault(kt["kind"], []).append(kt["ms"])
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    # kernels launched in the timed region: every step's graph, plus the device deal
    # (mandel_deal_lpt) of each sampled step of the N > 1 frame loop
    gpu_launches = kernels_per_step * args.steps
    if plan is not None:
        gpu_launches += sum(1 for k in range(plan_steps0, plan_steps0 + args.steps) if k % plan.sample_every == 0)
    # per-kernel breakdown (informational; outside the timed region): every kernel timed
    kall = {}
    for _ in range(3):
        step(timing=True)
        torch.cuda.synchronize()
        for kt in mb.kernel_times():
            kall.setdefault(kt["kind"], []).append(kt["ms"])
    my_total = sum(step_ms)
    total_ms = multigpu.max_over_ranks(my_total, device=cdev)
    exec_iters_all = multigpu.sum_over_ranks([float(exec_iters)], device=cdev)[0]
    tiles = plan.host_tiles() if plan is not None else None  # the deal of the last timed step
    ntiles = w.g * w.g if tiles is None else len(tiles)

    # ---- verification gather to rank 0 (N > 1 only; timed separately, not part of `value`)
    gather = None
    if world > 1 and not args.no_verify:
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        mb.ask(w.region, n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=tiles, scheme=args.scheme)
        parts = [None] * world
        dist.all_gather_object(parts, tiles)
        full = multigpu.gather_image(out if backend == "nccl" else out.cpu(), parts, w.g, rank)
        torch.cuda.synchronize()
        g_ms = 1e3 * (time.perf_counter() - t0)
        gather = {"ms": multigpu.max_over_ranks(g_ms, device=cdev), "backend": backend,
                  "bytes_to_rank0": 4 * (n * n - len(parts[0]) * (n // w.g) ** 2)}
        if rank == 0:
            ref = torch.empty_like(out)
            mb.ask(w.region, n, w.maxdwell, w.g, w.r, w.B, out=ref, scheme=args.scheme)
            gather["bit_exact_vs_1gpu_ask"] = bool(torch.equal(full.to(ref.device), ref))
            del ref
    ms_per_step = total_ms / args.steps
    value = n * n / (ms_per_step / 1e3) / 1e6  # Mpixel/s, whole job

    # ---- exhaustive baselines (same box, same image) and Σ dwell_Ex: the plain flat kernel
    # (the paper's Ex, escape test every 8 steps) and the tuned one (every 32 steps)
    extra = {}
    if rank == 0:
        ex_out = torch.empty((n, n), dtype=torch.int32, device=dev)
        ex_ms = {}
        for tuned in (False, True):
            mb.exhaustive(w.region, n, w.maxdwell, out=ex_out, tuned=tuned)
            torch.cuda.synchronize()
            ts = []
            for _ in range(2):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                mb.exhaustive(w.region, n, w.maxdwell, out=ex_out, tuned=tuned)
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ex_ms[tuned] = min(ts)
        sum_ex = int(ex_out.sum(dtype=torch.int64).item())
        if world == 1:
            mism = int((ex_out != out).sum().item())
            extra["mismatch_fraction_vs_exhaustive"] = mism / (n * n)
        del ex_out
        t_ex, t_ext = ex_ms[False], ex_ms[True]
        extra["exhaustive_ms"] = t_ex
        extra["exhaustive_tuned_ms"] = t_ext
        extra["exhaustive_giter_s"] = sum_ex / (t_ex / 1e3) / 1e9
        extra["exhaustive_tuned_giter_s"] = sum_ex / (t_ext / 1e3) / 1e9
        extra["exhaustive_sum_dwell"] = sum_ex
        extra["speedup_vs_exhaustive"] = t_ex / ms_per_step if world == 1 else None
        extra["speedup_vs_exhaustive_tuned"] = t_ext / ms_per_step if world == 1 else None
        extra["speedup_vs_exhaustive_1gpu"] = t_ex / ms_per_step
        extra["speedup_vs_exhaustive_tuned_1gpu"] = t_ext / ms_per_step
        extra["giter_s_effective"] = sum_ex / (ms_per_step / 1e3) / 1e9
    extra["giter_s_executed"] = exec_iters_all / (ms_per_step / 1e3) / 1e9

    # ---- e2e through the public API with host buffers (pinned), per step
    e2e = None
    if not args.no_e2e:
        # the 16-bit host image (mandel_ask_to_host_u16): dwells <= maxdwell <= 65535 are exact in
        # u16, and the copy -- the PCIe floor of this call -- carries half the bytes of int32
        h_out = torch.empty(n * n, dtype=torch.uint16).pin_memory()
        stage = torch.empty(n * n, dtype=torch.int16, device=out.device)
        mb.ask_to_host(w.region, n, w.maxdwell, w.g, w.r, w.B, h_out, out, ws, tiles=tiles, scheme=args.scheme,
                       stage=stage)
        e_ms = []
        if world > 1:
            dist.barrier()
        for _ in range(args.steps):
            t0 = time.perf_counter()
            mb.ask_to_host(w.region, n, w.maxdwell, w.g, w.r, w.B, h_out, out, ws, tiles=tiles,
                           scheme=args.scheme, stage=stage)
            e_ms.append(1e3 * (time.perf_counter() - t0))
        mine = sum(e_ms)
        if world > 1:
            tt = torch.tensor([mine], dtype=torch.float64, device=cdev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            mine = float(tt.item())
        e_step = mine / args.steps
        e2e = {"value": n * n / (e_step / 1e3) / 1e6, "unit": "Mpixel/s",
               "h2d_bytes_per_step": 4 * (0 if tiles is None else len(tiles)),
               "d2h_bytes_per_step": 2 * ntiles * (n // w.g) ** 2, "ms_per_step": e_step,
               "host_image": "uint16 (mandel_ask_to_host_u16)"}
        del h_out, stage

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (ALU-bound dwell loops).  peak = the MEASURED FP32
    # rate of the dwell step on this GPU (mandel_fp32_peak_probe: the 6-instruction step, no
    # escape test);
    # MEASURED_PEAKS.json has no FP32 entry.  The nominal 148 x 128 x f_max is reported beside.
    clocks = clk.summary()
    f_max = (clocks.get("sm_max_mhz") or 1965.0) * 1e6
    nominal = N_SM * LANES * f_max / 1e12  # T FP32 ops/s (one FADD/FMUL per lane per clock)
    measured = mb.fp32_peak_tops()
    peak_ops = measured if measured > 0 else nominal
    kt_sum = {k: sum(v) / args.steps for k, v in ktime.items()}         # live, timed region
    kt_launches = {k: len(v) / args.steps for k, v in ktime.items()}
    kt_all = {k: sum(v) / 3 for k, v in kall.items()}                   # breakdown, untimed
    dwell_kinds = {"b200_border": border_iters, "b200_leaf": leaf_iters, "sbr_level": border_iters,
                   "sbr_leaf": leaf_iters, "mbr_leaf": leaf_iters}
    dom = max((k for k in kt_sum if k in dwell_kinds), key=lambda k: kt_sum[k])
    achieved = FLOPS_PER_ITER * dwell_kinds[dom] / (kt_sum[dom] / 1e3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{args.workload}:{args.scheme}:{dom}")
        except (OSError, ValueError):
            traffic = None
    roofline = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak_ops, "unit": "TFLOP/s",
                "frac": achieved / peak_ops, "traffic": traffic,
                "peak_nominal": nominal, "frac_nominal": achieved / nominal,
                "launches_per_step": kt_launches[dom], "kernel_ms_per_step": kt_sum[dom],
                "frac_paper_7op": achieved * PAPER_OPS_PER_ITER / FLOPS_PER_ITER / peak_ops,
                "peak_basis": ("measured: mandel_fp32_peak_probe, the dwell step (3 FMUL + 2 FADD + 1 FFMA) on 2 "
                               "independent orbits per thread, 2048 threads/SM, no escape test (T FP32 lane-"
                               "instructions/s, FMUL/FADD/FFMA = 1 each); "
                               f"nominal {N_SM} SMs x {LANES} lanes x {f_max/1e6:.0f} MHz beside it; "
                               "6 FP32 instructions per dwell iteration executed (frac_paper_7op: the paper's "
                               "literal 7-op step count over the same peak)")}
    # border levels: the same algorithmic-ops / measured-peak fraction (all levels together)
    if "b200_border" in kt_all and kt_all["b200_border"] > 0:
        roofline["border_frac"] = FLOPS_PER_ITER * border_iters / (kt_all["b200_border"] / 1e3) / 1e12 / peak_ops
    for nm in ("exhaustive", "exhaustive_tuned"):  # the Ex kernels against the same measured peak
        if extra.get(nm + "_giter_s"):
            roofline[nm + "_frac"] = FLOPS_PER_ITER * extra[nm + "_giter_s"] / 1e3 / peak_ops
    pct_fp32 = 100.0 * FLOPS_PER_ITER * exec_iters_all / (ms_per_step / 1e3) / (2 * nominal * 1e12 * world)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_oracle_sample(w)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}

    # spread of this rank's per-step device times (mean +- stderr)
    sd = statistics.stdev(step_ms) if len(step_ms) > 1 else 0.0
    line = {"metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
            "ms_per_step_stderr": sd / math.sqrt(len(step_ms)), "ms_per_step_min": min(step_ms),
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config(w, args, world),
            "giter_s_effective": extra.get("giter_s_effective"),
            "giter_s_executed": extra["giter_s_executed"],
            "pct_fp32_peak_fma2": pct_fp32,
            "speedup_vs_exhaustive": extra.get("speedup_vs_exhaustive"),
            "speedup_vs_exhaustive_tuned": extra.get("speedup_vs_exhaustive_tuned"),
            "speedup_vs_exhaustive_1gpu": extra.get("speedup_vs_exhaustive_1gpu"),
            "speedup_vs_exhaustive_tuned_1gpu": extra.get("speedup_vs_exhaustive_tuned_1gpu"),
            "exhaustive_ms": extra.get("exhaustive_ms"),
            "exhaustive_tuned_ms": extra.get("exhaustive_tuned_ms"),
            "exhaustive_giter_s": extra.get("exhaustive_giter_s"),
            "exhaustive_tuned_giter_s": extra.get("exhaustive_tuned_giter_s"),
            "mismatch_fraction_vs_exhaustive": extra.get("mismatch_fraction_vs_exhaustive"),
            "executed_iters_per_step": exec_iters_all,
            "rank_tiles": ntiles,
            "verify_gather": gather,
            "kernel_ms_per_step": kt_all,
            "clocks": clocks, "e2e": e2e,
            "gpu_launches": gpu_launches,
            "roofline": roofline, "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
