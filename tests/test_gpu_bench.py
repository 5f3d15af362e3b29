"""bench.py end to end on the GPU (marked gpu): the N = 1 line's contract keys on the small C1
workload, and the N > 1 path -- two ranks over gloo sharing cuda:0, each running
multigpu.DevicePlan.step (sampled tile costs, side-stream all-reduce and device LPT deal one
step ahead) -- whose gathered image must equal the 1-GPU image bit for bit."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_single_gpu_c1():
    p = subprocess.run([sys.executable, "bench.py", "--workload", "C1", "--steps", "3", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    d = _last_json(p.stdout)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "Mpixel/s" and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "alu" and 0 < d["roofline"]["frac"] < 1.05
    assert d["e2e"]["d2h_bytes_per_step"] == 2 * 1024 * 1024  # 16-bit host image


def test_bench_two_ranks_gloo_c1():
    env = dict(os.environ, MANDEL_DIST_BACKEND="gloo")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", "C1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    d = _last_json(p.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["verify_gather"]["bit_exact_vs_1gpu_ask"] is True
    assert "side stream" in d["config"]["deal_plan"]
