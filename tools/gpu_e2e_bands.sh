# e2e (mandel_ask_to_host) time per band count at C3; parity of the banded path with each.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for NB in 4 8 16; do
  SO=$(python -c "
import sys; sys.path.insert(0, '.')
from paper_2206_02255_b200 import build
print(build.build(out='/tmp/libm_bands$NB.so', defines=['MANDEL_E2E_BANDS=$NB']))")
  MANDEL_B200_LIB=$SO timeout 300 python -c "
import time, torch, sys; sys.path.insert(0, '.')
import paper_2206_02255_b200 as mb, workloads as W
w = W.C3; n = w.n
out = torch.empty((n, n), dtype=torch.int32, device='cuda'); ws = mb.workspace(n, w.g, w.r, w.B)
h = torch.empty(n * n, dtype=torch.int32).pin_memory()
mb.ask_to_host(w.region, n, w.maxdwell, w.g, w.r, w.B, h, out, ws)
ts = []
for _ in range(6):
    t0 = time.perf_counter(); mb.ask_to_host(w.region, n, w.maxdwell, w.g, w.r, w.B, h, out, ws); ts.append(1e3 * (time.perf_counter() - t0))
ref = mb.ask(w.region, n, w.maxdwell, w.g, w.r, w.B).cpu().reshape(-1)
print('bands=$NB', 'e2e_ms min %.2f mean %.2f' % (min(ts), sum(ts) / len(ts)), 'same', bool(torch.equal(ref, h)))"
done
